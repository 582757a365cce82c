# round 2: A/B of the current build against experiment builds _exp/libl1rxg_<v>.so
# usage: bash tools/gpu_r2v.sh TAG v1 v2 ...   (segment tests on every build, 2 bench reps each, one parity line)
T=$1; shift
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched or persistent or attach or long_cn0" > gpurun_out/$T/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_seg.log
for v in "$@"; do
  L1RXG_SO=$PWD/_exp/libl1rxg_$v.so timeout 900 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched or persistent or attach or long_cn0" > gpurun_out/$T/pytest_seg_$v.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_seg_$v.log
done
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_main_$rep.json 2> gpurun_out/$T/b4_main_$rep.err
  for v in "$@"; do
    L1RXG_SO=$PWD/_exp/libl1rxg_$v.so timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_${v}_$rep.json 2> gpurun_out/$T/b4_${v}_$rep.err
  done
done
timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu-baseline > gpurun_out/$T/b4_parity.json 2> gpurun_out/$T/b4_parity.err
