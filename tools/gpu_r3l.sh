# r3l: latency shape with more work threads than runs (L1RXG_LAT_NWORK: phase B deals threads to taps): parity tests at 192, then configs 2/3/1 lines per setting
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
L1RXG_LAT_NWORK=192 timeout 600 python -m pytest tests/test_gpu_tracking.py -q -x -k "config1 or twelve or cluster_sizes or odd_epoch or multitap or monitor or real_if" > gpurun_out/$T/pytest_nw192.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_nw192.log
for NW in 0 128 192 256 384; do
for C in 2 3 1; do
  if [ $NW = 0 ]; then unset L1RXG_LAT_NWORK; else export L1RXG_LAT_NWORK=$NW; fi
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-companion > gpurun_out/$T/b${C}_nw$NW.json 2> gpurun_out/$T/b${C}_nw$NW.err
done
done
