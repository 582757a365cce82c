# First GPU pass of the segment correlator: gpurun --timeout 1800 -- "bash tools/gpu_seg1.sh"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/seg1
timeout 900 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched" > gpurun_out/seg1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/seg1/pytest.log
for cta in throughput segment; do
  timeout 600 python bench.py --config 4 --recordings 128 --blocks 100 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --cta $cta > gpurun_out/seg1/b4_$cta.json 2> gpurun_out/seg1/b4_$cta.err
done
