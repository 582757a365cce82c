# RUN-length A/B on the latency configs: gpurun -- "bash tools/gpu_run.sh tag testlib lib1 lib2 ..."
T=$1; TL=$2; shift; shift
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
L1RXG_SO=$PWD/$TL timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
for L in "$@"; do
  n=$(basename $L .so)
  for C in 2 3 1; do
    L1RXG_SO=$PWD/$L timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/b${C}_$n.json 2> gpurun_out/$T/b${C}_$n.err
  done
done
