T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_tracking.py -q -m gpu -x > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
for C in 1 2 3; do timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/b$C.json 2> gpurun_out/$T/b$C.err; done
