# parity + bench for each experiment build: gpurun -- "bash tools/gpu_abx.sh tag lib1 lib2 ..."
T=$1; shift
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
for L in "$@"; do
  n=$(basename $L .so)
  L1RXG_SO=$PWD/$L timeout 900 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched or persistent" > gpurun_out/$T/pytest_$n.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_$n.log
  L1RXG_SO=$PWD/$L timeout 600 python bench.py --config 4 --recordings 128 --blocks 100 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --cta segment > gpurun_out/$T/b4_$n.json 2> gpurun_out/$T/b4_$n.err
done
