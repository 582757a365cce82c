# r3c: RAW variant of the overlapped kernel (raw real-IF byte ring + FIR warps; L1RXG_OVL_RAWIF=0 = float2 ring + ingest pass):
# GPU tests, config 1/2 A/B with DRAM bytes; then segment-correlator pacing slack x work-item size at full size
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 600 python -m pytest tests/test_gpu_tracking.py -q -x > gpurun_out/$T/pytest_track.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_track.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
for i in 1 2; do
for C in 2 1; do
for X in 0 1; do
L1RXG_OVL_RAWIF=$X timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-companion > gpurun_out/$T/b${C}_raw${X}_$i.json 2> gpurun_out/$T/b${C}_raw${X}_$i.err
done
done
done
for X in 0 1; do
L1RXG_OVL_RAWIF=$X timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/$T/l2_raw$X.csv \
  python bench.py --config 2 --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu_l2_raw$X.log 2>&1
done
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-companion"
for CP in "32 2" "32 4" "32 8" "16 4" "16 8"; do
  set -- $CP
  L1RXG_SEG_CHUNK=$1 L1RXG_SEG_PACE=$2 timeout 600 $B > gpurun_out/$T/b4_chunk$1_pace$2.json 2> gpurun_out/$T/b4_chunk$1_pace$2.err
  L1RXG_SEG_CHUNK=$1 L1RXG_SEG_PACE=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:track_seg --csv --log-file gpurun_out/$T/l4_chunk$1_pace$2.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu_l4_chunk$1_pace$2.log 2>&1
done
