# round 2: per-tap fill / chains4 A/B (FFMA2 in all), tests, ncu of the default build
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
for rep in 1 2; do
for L in paper_1907_00463_b200/_lib/libl1rxg.so _exp/libl1rxg_flat.so _exp/libl1rxg_chains4.so; do
  n=$(basename $L .so)
  L1RXG_SO=$PWD/$L timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_${n}_$rep.json 2> gpurun_out/$T/b4_${n}_$rep.err
done; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_seg_kernel -c 1 -o gpurun_out/$T/seg_steady \
  python bench.py --recordings 64 --blocks 400 --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu.log 2>&1
