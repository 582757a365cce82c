# A/B of one experiment build against the default on the latency configs: bash tools/gpu_abso.sh TAG VARIANT  (_exp/libl1rxg_VARIANT.so)
T=$1; V=$2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
L1RXG_SO=$PWD/_exp/libl1rxg_$V.so timeout 600 python -m pytest tests/test_gpu_tracking.py -q -x -k "config1 or twelve or cluster_sizes or odd_epoch or multitap or monitor or real_if or latency_shape" > gpurun_out/$T/pytest_$V.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_$V.log
for i in 1 2; do
for C in 2 3 1; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-companion > gpurun_out/$T/b${C}_def_$i.json 2> gpurun_out/$T/b${C}_def_$i.err
  L1RXG_SO=$PWD/_exp/libl1rxg_$V.so timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-companion > gpurun_out/$T/b${C}_${V}_$i.json 2> gpurun_out/$T/b${C}_${V}_$i.err
done
done
