# overlapped latency kernel: GPU tests, then config 1-3 A/B (L1RXG_OVL=0 = track_kernel)
#   gpurun -- "bash tools/gpu_ovl.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 300 python -m pytest tests/test_gpu_tracking.py -q -m gpu -x -k "not simulator" > gpurun_out/$T/pytest_track.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_track.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
for R in 1 2; do
for C in 1 2 3; do
  for O in 0 1; do
    L1RXG_OVL=$O timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/b$C.o$O.r$R.json 2> gpurun_out/$T/b$C.o$O.r$R.err
  done
done
done
