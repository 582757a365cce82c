# r3b: segment correlator at FULL size (512 recordings x 1000 blocks): epochs per work item
# (L1RXG_SEG_CHUNK; default max_e/8 = 125) vs DRAM traffic and time; 6 CTAs/SM (qd6) and I2FP builds
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-companion"
for CH in 0 64 32 16; do
  if [ $CH = 0 ]; then unset L1RXG_SEG_CHUNK; else export L1RXG_SEG_CHUNK=$CH; fi
  timeout 600 $B > gpurun_out/$T/b4_chunk$CH.json 2> gpurun_out/$T/b4_chunk$CH.err
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:track_seg --csv --log-file gpurun_out/$T/l4_chunk$CH.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu_l4_chunk$CH.log 2>&1
done
unset L1RXG_SEG_CHUNK
for V in qd6 i2fp; do
  L1RXG_SO=$GRAFT_REPO_ROOT/_exp/libl1rxg_$V.so timeout 600 $B > gpurun_out/$T/b4_$V.json 2> gpurun_out/$T/b4_$V.err
  L1RXG_SEG_CHUNK=32 L1RXG_SO=$GRAFT_REPO_ROOT/_exp/libl1rxg_$V.so timeout 600 $B > gpurun_out/$T/b4_${V}_chunk32.json 2> gpurun_out/$T/b4_${V}_chunk32.err
done
