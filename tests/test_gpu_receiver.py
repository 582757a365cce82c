"""examples/gpu_receiver (C ABI only): cold start on the search grid, the
reference's peak rule and hand-off, and closed-loop tracking of a recording
streamed from disk.  Every visible satellite must
be detected (and no absent PRN), and must lock (test_tracking.cpp:403-429
criteria: lock ratio > 0.9, |Doppler error| < 5 Hz)."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1907_00463_b200 import abi, simsource as ss

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "examples", "_build", "gpu_receiver")


def test_gpu_receiver_cold_start_and_tracking(tmp_path):
    assert os.path.exists(BIN), "build with make -C examples (__graft_entry__.build does)"
    fs, ifz = 16.368e6, 4.092e6
    rng = np.random.default_rng(123)
    vis = [2, 9, 17, 30]
    svs = [ss.Sv(prn=p, cn0_dbhz=rng.uniform(44, 48), doppler_hz=rng.uniform(-4500, 4500),
                 delay_chips=rng.uniform(0, 1023)) for p in vis]
    raw = ss.synth(800, fs, svs, fmt="int8_real_if", if_hz=ifz, seed=124, device="cuda").cpu().numpy()
    path = tmp_path / "rec.bin"
    raw.tofile(path)
    out = subprocess.run([BIN, str(path), "int8_real_if", str(fs), str(ifz), "--acq-ms", "10",
                          "--chunk-ms", "100"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    chans = {x["prn"]: x for x in lines if "prn" in x}
    summary = [x["summary"] for x in lines if "summary" in x][0]
    assert sorted(chans) == vis, (sorted(chans), vis)
    assert summary["recording_ms"] == 800 and summary["real_time_factor"] > 1.0
    for sv in svs:
        ch = chans[sv.prn]
        assert ch["state"] == abi.TRACKING, ch
        assert ch["epochs"] >= 790
        assert ch["carrier_lock_ratio"] > 0.9, ch
        assert abs(ch["doppler_hz"] - sv.doppler_hz) < 5.0, ch


def _run(path, fs, ifz, *extra):
    out = subprocess.run([BIN, str(path), "int8_real_if", str(fs), str(ifz), "--acq-ms", "10", *extra],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    return {x["prn"]: x for x in lines if "prn" in x}, [x["summary"] for x in lines if "summary" in x][0]


def test_gpu_receiver_paced_overflow_accounting(tmp_path):
    """Paced mode mirrors the reference's producer (pipeline.hpp:388-404,
    samples.hpp:162-170): blocks are released at their stream time into a
    bounded queue; a block that finds the queue full is dropped and counted
    (overflow_count, degraded: never silent loss, :393-397).  A consumer
    that keeps up sees no overflow and locks; a consumer slower than real
    time (test hook --consumer-delay-ms) overflows, is marked degraded, and
    the sample accounting still covers the whole recording (the dropped
    blocks are replaced by zeros, not skipped)."""
    assert os.path.exists(BIN)
    fs, ifz = 16.368e6, 4.092e6
    svs = [ss.Sv(prn=p, cn0_dbhz=47.0, doppler_hz=d, delay_chips=dl)
           for p, d, dl in ((5, 1200.0, 300.5), (21, -2100.0, 812.25))]
    raw = ss.synth(600, fs, svs, fmt="int8_real_if", if_hz=ifz, seed=131, device="cuda").cpu().numpy()
    path = tmp_path / "rec.bin"
    raw.tofile(path)
    chans, summ = _run(path, fs, ifz, "--chunk-ms", "20", "--paced", "--queue", "4")
    assert summ["paced"] and summ["overflows"] == 0 and not summ["degraded"], summ
    assert summ["recording_ms"] == 600 and 0.8 < summ["real_time_factor"] < 1.2, summ
    assert sorted(chans) == [5, 21] and all(c["carrier_lock_ratio"] > 0.9 for c in chans.values())
    chans, summ = _run(path, fs, ifz, "--chunk-ms", "20", "--paced", "--queue", "2",
                       "--consumer-delay-ms", "60")
    assert summ["overflows"] > 0 and summ["degraded"], summ
    assert summ["recording_ms"] == 600, summ  # the timeline is complete (dropped blocks as zeros)
