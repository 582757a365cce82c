# steady-state ncu capture of the segment kernel: gpurun -- "bash tools/gpu_ncu2.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:track_seg -c 1 -o gpurun_out/$T/seg python bench.py --config 4 --recordings 64 --blocks 400 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --cta segment > gpurun_out/$T/ncu.log 2>&1
