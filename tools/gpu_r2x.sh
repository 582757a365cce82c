# r2x: baseline short config-4 line + steady-state ncu capture (source page) of the segment correlator
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 600 python bench.py --config 4 --recordings 128 --blocks 100 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --cta segment > gpurun_out/$T/b4_main.json 2> gpurun_out/$T/b4_main.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:track_seg -c 1 -o gpurun_out/$T/seg python bench.py --config 4 --recordings 64 --blocks 400 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-companion --no-parity --cta segment > gpurun_out/$T/ncu.log 2>&1
