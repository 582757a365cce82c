# Full measurement pass used for profiles/: gpurun --timeout 2400 -- "bash tools/gpu_full.sh"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/full
python bench.py --config 4 > gpurun_out/full/bench_config4.json 2> gpurun_out/full/bench_config4.err
python bench.py --config 5 > gpurun_out/full/bench_config5.json 2> gpurun_out/full/bench_config5.err
python bench.py > gpurun_out/full/bench_config2.json 2> gpurun_out/full/bench_config2.err
KR='regex:"track_kernel|ingest_if4|decode_i|grid_fold|grid_corr|mix_generic|fir_generic"'
eval ncu --metrics gpu__time_duration.sum --clock-control none -k $KR -c 400 --csv --log-file gpurun_out/full/launches_config4.csv python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:track_kernel -c 1 -o gpurun_out/full/track_config4 python bench.py --config 4 --recordings 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:nvjet -c 1 -o gpurun_out/full/gemm_config5 python bench.py --config 5 --steps 1 --warmup 1 > /dev/null 2>&1
ls gpurun_out/full
