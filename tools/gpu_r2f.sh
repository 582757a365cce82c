# round 2: FFMA2 anchor/combine + quarter-grid start chips; A/B vs taploop1 and the exact start-chip path
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched or persistent or attach" > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_main_$rep.json 2> gpurun_out/$T/b4_main_$rep.err
  L1RXG_SEG_QGRID=0 timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_noq_$rep.json 2> gpurun_out/$T/b4_noq_$rep.err
  L1RXG_SO=$PWD/_exp/libl1rxg_taploop1.so timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_taploop1_$rep.json 2> gpurun_out/$T/b4_taploop1_$rep.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_seg_kernel -c 1 -o gpurun_out/$T/seg_steady \
  python bench.py --recordings 64 --blocks 400 --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu.log 2>&1
