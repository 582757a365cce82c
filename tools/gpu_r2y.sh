# r2y: segment-correlator tests + short config-4 lines, direct quarter-crossing kernel vs the step-table kernel
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched or persistent or quarter" > gpurun_out/$T/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_seg.log
for i in 1 2; do
timeout 600 python bench.py --config 4 --recordings 128 --blocks 100 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --cta segment > gpurun_out/$T/b4_qd_$i.json 2> gpurun_out/$T/b4_qd_$i.err
L1RXG_SEG_QDIRECT=0 timeout 600 python bench.py --config 4 --recordings 128 --blocks 100 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --cta segment > gpurun_out/$T/b4_tab_$i.json 2> gpurun_out/$T/b4_tab_$i.err
done
