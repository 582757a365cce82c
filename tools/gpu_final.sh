# final pass: gpurun -- "bash tools/gpu_final.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$T/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/$T/smoke.log
timeout 900 python bench.py > gpurun_out/$T/bench_default.json 2> gpurun_out/$T/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/$T/ref_default.json 2> gpurun_out/$T/ref_default.err
for C in 1 3 4 5; do
  timeout 900 python bench.py --config $C > gpurun_out/$T/bench_config$C.json 2> gpurun_out/$T/bench_config$C.err
done
timeout 600 python bench.py --impl reference --config 4 > gpurun_out/$T/ref_config4.json 2> gpurun_out/$T/ref_config4.err
