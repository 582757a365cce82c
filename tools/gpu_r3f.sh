# r3f: gang tickets by warp-slot class (default) vs the single item queue (L1RXG_SEG_GANGS=0), full size, per work-item size;
# DRAM bytes per launch; segment tests
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 400 python -m pytest tests/test_gpu_tracking.py tests/test_gpu_baseline_sizes.py -q -x -k "segment or batched or persistent or quarter or config4 or wideband" > gpurun_out/$T/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_seg.log
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-companion"
for CH in 32 16 64; do
for G in 1 0; do
  L1RXG_SEG_GANGS=$G L1RXG_SEG_CHUNK=$CH timeout 400 $B > gpurun_out/$T/b4_chunk${CH}_g$G.json 2> gpurun_out/$T/b4_chunk${CH}_g$G.err
done
  L1RXG_SEG_CHUNK=$CH timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:track_seg --csv --log-file gpurun_out/$T/l4_chunk${CH}_g1.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu_l4_chunk${CH}_g1.log 2>&1
done
L1RXG_SEG_CHUNK=32 L1RXG_SEG_TRACE=/tmp/segtrace.txt timeout 400 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-companion --no-parity > gpurun_out/$T/trace_run.json 2> gpurun_out/$T/trace_run.err
python tools/seg_trace_stats.py /tmp/segtrace.txt > gpurun_out/$T/trace_stats_chunk32.txt 2>&1
