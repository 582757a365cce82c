cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/full
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"track_kernel|ingest_if4|decode_iq|grid_fold|grid_corr|mix_generic|fir_generic" -c 400 --csv --log-file gpurun_out/full/launches_config4.csv python bench.py --config 4 --recordings 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/full/*.csv
