# round 2: tests, default bench (config 4 headline), reference arm, cluster A/B
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 900 python bench.py > gpurun_out/$T/bench_default.json 2> gpurun_out/$T/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/$T/ref_default.json 2> gpurun_out/$T/ref_default.err
for C in 4 9; do for K in auto 8 16; do
  if [ $K = auto ]; then timeout 120 python tools/cluster_ab.py $C >> gpurun_out/$T/cluster_ab.txt 2>&1
  else L1RXG_CLUSTER=$K timeout 120 python tools/cluster_ab.py $C >> gpurun_out/$T/cluster_ab.txt 2>&1; fi
done; done
