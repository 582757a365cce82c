# quick check of a build: full GPU tests, smoke, the default line and the config-2 line: gpurun -- "bash tools/gpu_check.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$T/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/$T/smoke.log
timeout 900 python bench.py > gpurun_out/$T/bench_default.json 2> gpurun_out/$T/bench_default.err
timeout 600 python bench.py --config 2 > gpurun_out/$T/bench_config2.json 2> gpurun_out/$T/bench_config2.err
