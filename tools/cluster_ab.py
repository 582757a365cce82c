"""Cluster-size A/B for the latency shape (the auto rule's
16-CTA clusters): C channels on one int8 real-IF stream at 16.368 MHz, E/P/L,
`blocks` epochs; prints the tracking ms per launch (median of 3).
    L1RXG_CLUSTER=K python tools/cluster_ab.py C [blocks]"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_00463_b200 import abi, simsource as ss  # noqa: E402
from paper_1907_00463_b200.tracking import Context, Tracker, init_channel_from_acquisition  # noqa: E402

C = int(sys.argv[1])
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
fs, ifz, n = 16.368e6, 4.092e6, 16368
rng = np.random.default_rng(7)
svs = [ss.Sv(prn=p, cn0_dbhz=45.0, doppler_hz=rng.uniform(-4000, 4000), delay_chips=rng.uniform(0, 1023))
       for p in range(1, C + 1)]
raw = ss.synth(blocks, fs, svs, fmt="int8_real_if", if_hz=ifz, seed=3, device="cuda")
inits = []
for sv in svs:
    b, d = ss.truth_channel_start(sv, fs)
    inits.append(init_channel_from_acquisition(sv.prn, d, 0, b, 0, fs))
cfg = abi.TrackingCfg.default()
cfg.lock_fail_limit = 2**31 - 1
ctx = Context(0)
trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, fs, ifz, inits, cfg=cfg, ring_samples=(blocks + 8) * n,
              max_records=blocks)
ms = []
for rep in range(4):
    trk.reset(inits)
    trk.push_device(0, raw.data_ptr(), raw.numel())
    trk.run()
    trk.sync()
    _, t, _ = trk.timing()
    if rep:
        ms.append(t)
print("C=%d K=%s track_ms=%.3f epochs=%d" % (C, os.environ.get("L1RXG_CLUSTER", "auto"), statistics.median(ms),
                                              int(trk.epoch_counts().min())))
