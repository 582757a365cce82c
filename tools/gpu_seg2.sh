# Segment correlator: parity + one ncu capture: gpurun --timeout 1800 -- "bash tools/gpu_seg2.sh"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/seg2
timeout 900 python -m pytest tests/test_gpu_tracking.py -q -k "segment or batched" > gpurun_out/seg2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/seg2/pytest.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_seg -c 1 -o gpurun_out/seg2/seg python bench.py --config 4 --recordings 64 --blocks 50 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --cta segment > gpurun_out/seg2/ncu.log 2>&1
ls -la gpurun_out/seg2
