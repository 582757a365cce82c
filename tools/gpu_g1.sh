cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1/smi.txt
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/g1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g1/smoke.log
timeout 900 python bench.py > gpurun_out/g1/bench2.json 2> gpurun_out/g1/bench2.err; echo "rc=$?" >> gpurun_out/g1/bench2.err
timeout 1200 python bench.py --config 4 > gpurun_out/g1/bench4.json 2> gpurun_out/g1/bench4.err; echo "rc=$?" >> gpurun_out/g1/bench4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g1/ref2.json 2> gpurun_out/g1/ref2.err
