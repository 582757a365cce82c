# ncu of the overlapped latency kernel on config 2: gpurun -- "bash tools/gpu_ncu_ovl.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$T/launches_config2.csv python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/ncu_launches.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:track_ovl -c 1 -o gpurun_out/$T/ovl python bench.py --config 2 --blocks 2000 --steps 1 --warmup 1 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/ncu_full.log 2>&1
