# r3d: sibling spread of the segment correlator's work items at full size (L1RXG_SEG_TRACE), per work-item size;
# then full-size lines with the cheaper item start (parallel state copy, per-context chip words)
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 600 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched or persistent or quarter" > gpurun_out/$T/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_seg.log
for CH in 0 32 16; do
  if [ $CH = 0 ]; then unset L1RXG_SEG_CHUNK; else export L1RXG_SEG_CHUNK=$CH; fi
  L1RXG_SEG_TRACE=/tmp/segtrace_$CH.txt timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-companion --no-parity > gpurun_out/$T/trace_run_$CH.json 2> gpurun_out/$T/trace_run_$CH.err
  python tools/seg_trace_stats.py /tmp/segtrace_$CH.txt > gpurun_out/$T/trace_stats_chunk$CH.txt 2>&1
  head -2000 /tmp/segtrace_$CH.txt > gpurun_out/$T/trace_head_chunk$CH.txt
done
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-companion"
for CH in 32 16 8; do
  L1RXG_SEG_CHUNK=$CH timeout 600 $B > gpurun_out/$T/b4_chunk$CH.json 2> gpurun_out/$T/b4_chunk$CH.err
done
