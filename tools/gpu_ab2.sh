# full GPU tests (in-tree build) + config-2 A/B: gpurun -- "bash tools/gpu_ab2.sh tag lib1 lib2 ..."
T=$1; shift
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
for L in "$@"; do
  n=$(basename $L .so)
  L1RXG_SO=$PWD/$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-companion > gpurun_out/$T/b2_$n.json 2> gpurun_out/$T/b2_$n.err
done
