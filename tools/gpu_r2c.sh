# round 2: FFMA2 run loop -- tests, config-4 value, steady-state ncu capture, cluster A/B 6/8 channels
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 600 python bench.py --no-e2e --no-companion --no-cpu-baseline > gpurun_out/$T/bench_config4.json 2> gpurun_out/$T/bench_config4.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_seg_kernel -c 1 -o gpurun_out/$T/seg_steady \
  python bench.py --recordings 64 --blocks 400 --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu.log 2>&1
for C in 6 8; do for K in 8 16; do
  L1RXG_CLUSTER=$K timeout 120 python tools/cluster_ab.py $C >> gpurun_out/$T/cluster_ab.txt 2>&1
done; done
