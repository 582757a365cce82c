# full pass: gpurun -- "bash tools/gpu_pass.sh tag" (tests, smoke, default bench + reference arm, configs 1/2/3/5, ncu of the hot kernels)
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$T/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/$T/smoke.log
timeout 900 python bench.py > gpurun_out/$T/bench_default.json 2> gpurun_out/$T/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/$T/ref_default.json 2> gpurun_out/$T/ref_default.err
for C in 5 2 1 3; do
  timeout 900 python bench.py --config $C > gpurun_out/$T/bench_config$C.json 2> gpurun_out/$T/bench_config$C.err
done
timeout 600 python bench.py --config 5 --impl reference > gpurun_out/$T/ref_config5.json 2> gpurun_out/$T/ref_config5.err
timeout 600 python bench.py --config 2 --impl reference > gpurun_out/$T/ref_config2.json 2> gpurun_out/$T/ref_config2.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:grid_mma_kernel -c 1 -o gpurun_out/$T/grid_mma \
  python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/$T/ncu_grid.log 2>&1
# (gpurun brings back at most 64 MiB: keep the raw page of this report, not the report)
ncu -i gpurun_out/$T/grid_mma.ncu-rep --page raw --csv > gpurun_out/$T/grid_mma_raw.csv 2>/dev/null && rm -f gpurun_out/$T/grid_mma.ncu-rep
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$T/launches5.csv \
  python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/$T/ncu_l5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_seg_kernel -c 1 -o gpurun_out/$T/seg_steady \
  python bench.py --recordings 64 --blocks 400 --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu_seg.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/$T/launches4.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu_l4.log 2>&1
