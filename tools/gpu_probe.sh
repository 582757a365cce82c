# box probe + current-state check: gpurun -- "bash tools/gpu_probe.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
{ free -g; nproc; lscpu | grep -E 'Model name|Socket|Thread|Core|NUMA'; nvidia-smi; df -h /dev/shm; ulimit -l; } > gpurun_out/$T/box.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 900 python bench.py --config 4 > gpurun_out/$T/bench_config4.json 2> gpurun_out/$T/bench_config4.err
