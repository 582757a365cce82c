# r3a: gang pacing of the segment correlator (L1RXG_SEG_PACE 0/1/2) and the direct cluster exchange of the
# overlapped latency kernel (L1RXG_OVL_XD 0/1): tracking tests, then short A/B lines
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 1200 python -m pytest tests/test_gpu_tracking.py tests/test_gpu_baseline_sizes.py -q -x > gpurun_out/$T/pytest_track.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_track.log
for i in 1 2; do
for P in 0 1 2; do
L1RXG_SEG_PACE=$P timeout 600 python bench.py --config 4 --recordings 128 --blocks 200 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-companion --cta segment > gpurun_out/$T/b4_pace${P}_$i.json 2> gpurun_out/$T/b4_pace${P}_$i.err
done
for C in 2 1 3; do
for X in 0 1; do
L1RXG_OVL_XD=$X timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/b${C}_xd${X}_$i.json 2> gpurun_out/$T/b${C}_xd${X}_$i.err
done
done
done
for P in 0 1; do
L1RXG_SEG_PACE=$P timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:track_seg --csv --log-file gpurun_out/$T/l4_pace$P.csv \
  python bench.py --config 4 --recordings 128 --blocks 200 --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity --cta segment > gpurun_out/$T/ncu_l4_pace$P.log 2>&1
done
