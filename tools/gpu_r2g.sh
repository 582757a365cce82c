# round 2: K4c (tcgen05 int8 grid kernel) -- search tests, config-5 bench per path, ncu of grid_mma_kernel
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 600 python -m pytest tests/test_gpu_search.py tests/test_gpu_coldstart.py -q -x > gpurun_out/$T/pytest_search.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_search.log
for P in mma gemm fp32; do
  L1RXG_GRID=$P timeout 300 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/$T/b5_$P.json 2> gpurun_out/$T/b5_$P.err
done
timeout 300 python bench.py --config 5 --impl reference --steps 2 --warmup 1 > gpurun_out/$T/ref5.json 2> gpurun_out/$T/ref5.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:grid_mma_kernel -c 1 -o gpurun_out/$T/grid_mma \
  python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/$T/ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$T/launches5.csv \
  python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/$T/ncu_l.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
