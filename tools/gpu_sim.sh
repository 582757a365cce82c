# simulator tests: gpurun -- "bash tools/gpu_sim.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 600 python -m pytest tests/test_gpu_tracking.py -q -k "simulator" > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
timeout 300 python -c "
import time, torch
from paper_1907_00463_b200 import simsource as ss
from paper_1907_00463_b200.tracking import Context
ctx = Context(0)
recs = [[ss.Sv(prn=p, cn0_dbhz=40.0, doppler_hz=100.0*p, delay_chips=10.0*p) for p in range(1, 13)] for r in range(64)]
out = ss.synth_gpu(ctx, 100, 65.472e6, recs)
torch.cuda.synchronize(); t = time.perf_counter()
out = ss.synth_gpu(ctx, 100, 65.472e6, recs, out=out)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print('simulate 64 rec x 100 ms x 12 SV at 65.472 MHz: %.3f s, %.1f GB/s of cint16' % (dt, out.numel() / dt / 1e9))
" > gpurun_out/$T/speed.log 2>&1
