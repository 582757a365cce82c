# r3e: (1) item durations by warp slot / SM (scheduler fairness diagnostic); (2) RAW variant with the register-blocked FIR: config 1/2 A/B, NF=2 build
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
L1RXG_SEG_CHUNK=32 L1RXG_SEG_TRACE=/tmp/segtrace.txt timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-companion --no-parity > gpurun_out/$T/trace_run.json 2> gpurun_out/$T/trace_run.err
python tools/seg_trace_stats.py /tmp/segtrace.txt > gpurun_out/$T/trace_stats_chunk32.txt 2>&1
head -3000 /tmp/segtrace.txt > gpurun_out/$T/trace_head_chunk32.txt
timeout 300 python -m pytest tests/test_gpu_tracking.py -q -x -k "real_if or config1 or twelve or cluster_sizes or latency_shape" > gpurun_out/$T/pytest_raw.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_raw.log
for i in 1 2; do
for C in 2 1; do
L1RXG_OVL_RAWIF=0 timeout 300 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-companion > gpurun_out/$T/b${C}_raw0_$i.json 2> gpurun_out/$T/b${C}_raw0_$i.err
timeout 300 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-companion > gpurun_out/$T/b${C}_raw1_$i.json 2> gpurun_out/$T/b${C}_raw1_$i.err
L1RXG_SO=$GRAFT_REPO_ROOT/_exp/libl1rxg_nf2.so timeout 300 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-companion > gpurun_out/$T/b${C}_nf2_$i.json 2> gpurun_out/$T/b${C}_nf2_$i.err
done
done
