# round 2: LDS tap combine A/B; search grid ex + config 5 e2e; search/receiver tests
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_receiver.py tests/test_gpu_coldstart.py -q > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 900 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched or persistent or attach" > gpurun_out/$T/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_seg.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_lds_$rep.json 2> gpurun_out/$T/b4_lds_$rep.err
  L1RXG_SO=$PWD/_exp/libl1rxg_selcomb.so timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/b4_sel_$rep.json 2> gpurun_out/$T/b4_sel_$rep.err
done
timeout 300 python bench.py --config 5 > gpurun_out/$T/bench_config5.json 2> gpurun_out/$T/bench_config5.err
