# Demo: 5 s / 12-SV recording through examples/_build/gpu_receiver, free-running and paced.
cd $GRAFT_REPO_ROOT
python - <<'PY'
import numpy as np
from paper_1907_00463_b200 import simsource as ss
rng = np.random.default_rng(5)
svs = [ss.Sv(prn=p, cn0_dbhz=rng.uniform(40, 48), doppler_hz=rng.uniform(-4500, 4500), delay_chips=rng.uniform(0, 1023)) for p in (1,4,7,11,13,17,20,23,26,29,31,32)]
raw = ss.synth(5000, 16.368e6, svs, fmt="int8_real_if", if_hz=4.092e6, seed=6, device="cuda").cpu().numpy()
raw.tofile("/tmp/rec12.bin")
PY
./examples/_build/gpu_receiver /tmp/rec12.bin int8_real_if 16368000 4092000 --acq-ms 10 --chunk-ms 500 | tail -1
./examples/_build/gpu_receiver /tmp/rec12.bin int8_real_if 16368000 4092000 --acq-ms 10 --chunk-ms 100 --paced --max-ms 2000 | tail -1
