# r3k: vectorised ingest_if4_kernel (four outputs per thread from registers, 16-byte ring stores): ingest/search tests, configs 2/1/5 lines
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 600 python -m pytest tests/test_gpu_tracking.py tests/test_gpu_search.py tests/test_gpu_coldstart.py -q -x -k "ingest or config1 or twelve or real_if or search or cold or grid" > gpurun_out/$T/pytest_ingest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_ingest.log
for C in 2 1 5; do
  timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/$T/bench_config$C.json 2> gpurun_out/$T/bench_config$C.err
done
