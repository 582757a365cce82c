# r3i: after removing the pacing / direct-exchange experiment code: full GPU tests, default line, config 2 line,
# and a representative steady-state ncu capture of the segment correlator with the gang tickets (256 recordings x 96 blocks)
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$T/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/$T/smoke.log
timeout 900 python bench.py > gpurun_out/$T/bench_default.json 2> gpurun_out/$T/bench_default.err
timeout 600 python bench.py --config 2 > gpurun_out/$T/bench_config2.json 2> gpurun_out/$T/bench_config2.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_seg_kernel -c 1 -o gpurun_out/$T/seg_steady \
  python bench.py --recordings 256 --blocks 96 --steps 1 --warmup 1 --no-e2e --no-companion --no-cpu-baseline --no-parity > gpurun_out/$T/ncu_seg.log 2>&1
