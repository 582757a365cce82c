# seg iteration incl. attach: gpurun --timeout 1800 -- "bash tools/gpu_seg6.sh tag"
T=${1:-seg6}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_tracking.py -q -x -k "segment or batched" > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
for cta in throughput segment; do
  timeout 600 python bench.py --config 4 --recordings 128 --blocks 100 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --cta $cta > gpurun_out/$T/b4_$cta.json 2> gpurun_out/$T/b4_$cta.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_seg -c 1 -o gpurun_out/$T/seg python bench.py --config 4 --recordings 64 --blocks 50 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --cta segment > gpurun_out/$T/ncu.log 2>&1
