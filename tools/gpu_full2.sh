# Full measurement pass (round 1, session 2): gpurun --timeout 3000 -- "bash tools/gpu_full2.sh"
cd $GRAFT_REPO_ROOT; T=${1:-full2}; mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$T/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/$T/smoke.log
timeout 900 python bench.py --config 4 > gpurun_out/$T/bench_config4.json 2> gpurun_out/$T/bench_config4.err
timeout 900 python bench.py > gpurun_out/$T/bench_config2.json 2> gpurun_out/$T/bench_config2.err
timeout 600 python bench.py --impl reference --config 4 --steps 3 --warmup 3 > gpurun_out/$T/ref_config4.json 2> gpurun_out/$T/ref_config4.err
KR='regex:"track_seg|track_kernel|ingest_if4|decode_i|copy_raw|grid_fold|grid_corr"'
eval timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k $KR -c 50 --csv --log-file gpurun_out/$T/launches_config4.csv python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_seg -c 1 -o gpurun_out/$T/seg_config4 python bench.py --config 4 --recordings 64 --blocks 50 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls gpurun_out/$T
