# ncu capture of the config-2 latency kernel: gpurun -- "bash tools/gpu_ncu_c2.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_kernel -c 1 -o gpurun_out/$T/c2 python bench.py --blocks 2000 --steps 1 --warmup 1 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/ncu.log 2>&1
