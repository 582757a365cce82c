# launch list of the repo's own kernels on config 2: gpurun -- "bash tools/gpu_launch2.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"track|ingest|simgen|grid_corr|correlate" -c 200 --csv --log-file gpurun_out/$T/launches_config2.csv python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/ncu_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"track|ingest|simgen|grid_corr|correlate" -c 200 --csv --log-file gpurun_out/$T/launches_config3.csv python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/ncu_launches3.log 2>&1
