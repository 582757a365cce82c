# round 2: 32-bit barrier addresses + fix-up addressing vs the previous build
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched or persistent or attach or long_cn0" > gpurun_out/$T/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_seg.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_main_$rep.json 2> gpurun_out/$T/b4_main_$rep.err
  L1RXG_SO=$PWD/_exp/libl1rxg_prev.so timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_prev_$rep.json 2> gpurun_out/$T/b4_prev_$rep.err
done
timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu-baseline > gpurun_out/$T/b4_parity.json 2> gpurun_out/$T/b4_parity.err
