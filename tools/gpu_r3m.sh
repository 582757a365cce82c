# r3m: the measured work-thread rule in place (config 2: 192, config 3: 128): tracking tests, then neighbours of the rule
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_tracking.py tests/test_gpu_baseline_sizes.py tests/test_gpu_adapter.py -q -x > gpurun_out/$T/pytest_track.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_track.log
for NW in rule 160 224; do
  if [ $NW = rule ]; then unset L1RXG_LAT_NWORK; else export L1RXG_LAT_NWORK=$NW; fi
  timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-companion > gpurun_out/$T/b2_nw$NW.json 2> gpurun_out/$T/b2_nw$NW.err
done
for NW in rule 160; do
  if [ $NW = rule ]; then unset L1RXG_LAT_NWORK; else export L1RXG_LAT_NWORK=$NW; fi
  timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-companion > gpurun_out/$T/b3_nw$NW.json 2> gpurun_out/$T/b3_nw$NW.err
done
unset L1RXG_LAT_NWORK
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-companion > gpurun_out/$T/b1_nwrule.json 2> gpurun_out/$T/b1_nwrule.err
