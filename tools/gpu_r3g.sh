# r3g: new defaults (gang tickets, 16-epoch items) vs the 6-CTAs-per-SM build (qd6), full size, twice each; DRAM bytes for both
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-companion"
for i in 1 2; do
  timeout 400 $B > gpurun_out/$T/b4_def_$i.json 2> gpurun_out/$T/b4_def_$i.err
  L1RXG_SO=$GRAFT_REPO_ROOT/_exp/libl1rxg_qd6.so timeout 400 $B > gpurun_out/$T/b4_qd6_$i.json 2> gpurun_out/$T/b4_qd6_$i.err
done
L1RXG_SO=$GRAFT_REPO_ROOT/_exp/libl1rxg_qd6.so timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:track_seg --csv --log-file gpurun_out/$T/l4_qd6.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu_l4_qd6.log 2>&1
L1RXG_SO=$GRAFT_REPO_ROOT/_exp/libl1rxg_qd6.so timeout 400 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched or persistent or quarter" > gpurun_out/$T/pytest_seg_qd6.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_seg_qd6.log
