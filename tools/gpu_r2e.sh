# round 2: tests (per-thread per-call streams, acquisition pins, full-shape parity), fill/ILP A/B
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
for rep in 1 2; do
for L in _exp/libl1rxg_flat.so _exp/libl1rxg_taploop1.so _exp/libl1rxg_split2.so; do
  n=$(basename $L .so)
  L1RXG_SO=$PWD/$L timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_${n}_$rep.json 2> gpurun_out/$T/b4_${n}_$rep.err
done; done
