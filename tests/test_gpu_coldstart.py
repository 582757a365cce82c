"""GPU cold start: the search grid's detections are
handed to the tracker, which must pull in and lock on every visible
satellite (the reference's closed-loop criteria, test_tracking.cpp:403-429:
lock ratio > 0.9, |Doppler error| < 5 Hz), and absent PRNs must not be
detected."""
import numpy as np
import pytest

from paper_1907_00463_b200 import abi, simsource as ss
from paper_1907_00463_b200.coldstart import acquire, handoff
from paper_1907_00463_b200.tracking import Tracker

pytestmark = pytest.mark.gpu


def test_grid_detections_hand_off_to_tracking(ctx):
    fs, ifz, n = 16.368e6, 4.092e6, 16368
    rng = np.random.default_rng(77)
    vis = [3, 11, 19, 26]
    svs = [ss.Sv(prn=p, cn0_dbhz=rng.uniform(44, 48), doppler_hz=rng.uniform(-4500, 4500),
                 delay_chips=rng.uniform(0, 1023)) for p in vis]
    ms = 700
    raw = ss.synth(ms, fs, svs, fmt="int8_real_if", if_hz=ifz, seed=78, device="cuda")
    bins = np.arange(-5000.0, 5000.1, 500.0)
    res, _ = acquire(ctx, raw.numel(), abi.FMT_INT8_REAL_IF, fs, ifz, 10, np.arange(1, 33), bins,
                     device_ptr=raw.data_ptr())
    det = {r.prn: r for r in res if r.detected}
    assert set(vis) <= set(det), (sorted(det), vis)
    assert set(det) == set(vis), "false detections: %s" % sorted(set(det) - set(vis))
    chans = handoff([det[p] for p in vis], fs)
    trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, fs, ifz, chans, ring_samples=(ms + 8) * n,
                  max_records=ms)
    trk.push_device(0, raw.data_ptr(), raw.numel())
    trk.run()
    for c, sv in enumerate(svs):
        rec = trk.records(c)
        assert len(rec) >= ms - 5
        tail = rec[-100:]
        assert float(np.median(tail["carrier_lock_ratio"])) > 0.9, sv
        assert abs(float(np.median(tail["carrier_doppler_hz"])) - sv.doppler_hz) < 5.0, sv
        assert int(tail["state"][-1]) != abi.IDLE
