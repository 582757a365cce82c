"""Parity at BASELINE.json's full shapes (VERDICT r1 "missing 6"; the
reference's own analogue is the 200-epoch kernel equivalence of
test_tracking.cpp:166-204): the exact bench scenarios (bench.py scenario(),
same seeds and channel maps) of config 2 (12 channels, int8 real IF) and
config 3 (32 channels x 13 taps, cint16, 8 authentic + 8 spoofed PRNs) over
2 000 1-ms blocks through the default latency kernels, every channel's
epochs replayed by the oracle from the GPU's own pre-state on a
deterministic sample (all epochs of channel 0, every 7th epoch of the
others) -- sums within 1e-5 x max|E/P/L| (and every tap), NCO advance
bit-exact, loop outputs within 1e-5.  Config 4's full size (512 recordings x
1 000 blocks) is replayed inside bench.py's default line (parity field);
config 5's full grid against the reference plane below."""
import numpy as np
import pytest

import bench
from paper_1907_00463_b200 import abi, simsource as ss
from paper_1907_00463_b200.tracking import Tracker, search_grid

pytestmark = pytest.mark.gpu

BLOCKS = 2000


@pytest.mark.parametrize("cfg_id", [2, 3])
def test_full_shape_replay(ctx, oracle_mod, cfg_id):
    from oracle.replay import replay_sampled
    c, svs, chans = bench.scenario(cfg_id, bench.CONFIGS[cfg_id]["seed"])
    fs, n = c["fs"], int(round(c["fs"] / 1000))
    taps = bench.make_taps(c["taps"])
    cfg = abi.TrackingCfg.default()
    cfg.lock_fail_limit = 2**31 - 1
    inits = bench.channel_inits(chans, fs)
    raw = ss.synth(BLOCKS, fs, svs, fmt=c["fmt"], if_hz=c["if_hz"], seed=c["seed"], device="cuda")
    fmt = {"int8_real_if": abi.FMT_INT8_REAL_IF, "int16_iq": abi.FMT_INT16_IQ}[c["fmt"]]
    trk = Tracker(ctx, fmt, fs, c["if_hz"], inits, taps=taps, cfg=cfg, ring_samples=(BLOCKS + 8) * n,
                  max_records=BLOCKS)
    trk.push_device(0, raw.data_ptr(), raw.numel())
    trk.run()
    counts = trk.epoch_counts()
    assert len(counts) == len(chans) and counts.min() >= BLOCKS - 2
    x = oracle_mod.ingest(raw.cpu().numpy(), fmt, fs, c["if_hz"])
    r0 = replay_sampled(oracle_mod, trk, [0], inits, lambda _: x, n, cfg, taps, fs, every=1)
    rs = replay_sampled(oracle_mod, trk, list(range(1, len(chans))), inits, lambda _: x, n, cfg, taps, fs,
                        every=7)
    print(cfg_id, r0, rs)
    for r in (r0, rs):
        assert r["mismatches"] == 0, r["first_mismatch"]
        assert r["worst"]["sums"] <= 1e-5 and r["worst"]["taps"] <= 1e-5 and r["worst"]["loop"] <= 1e-5, r
    assert r0["checked"] + rs["checked"] >= BLOCKS + (len(chans) - 1) * (BLOCKS - 2) // 7


def test_config5_full_grid_against_reference_plane(ctx, oracle_mod):
    """Config 5 at full size (PRNs 1-32 x 41 bins x 2 046 delays x 20 blocks,
    the bench scenario): the GPU plane of two present PRNs and one absent one
    equals the reference acquire_pcs plane (acquisition.hpp over cuFFTW) on
    the half-chip delays at three bins each, within 1e-5 of the largest cell."""
    if not oracle_mod.acq_available():
        pytest.skip("reference acquisition shim not built")
    g = bench.GRID
    rng = np.random.default_rng(g["seed"])
    prns_sv = rng.choice(np.arange(1, 33), 6, replace=False)
    svs = [ss.Sv(prn=int(p), cn0_dbhz=rng.uniform(25, 45), doppler_hz=rng.uniform(-9000, 9000),
                 delay_chips=rng.uniform(0, 1023)) for p in prns_sv]
    fs, N, blocks = g["fs"], 16368, g["blocks"]
    raw = ss.synth(blocks, fs, svs, fmt="int8_real_if", if_hz=g["if_hz"], seed=g["seed"], device="cuda")
    bins = g["bins"]
    plane = search_grid(ctx, raw.numel(), abi.FMT_INT8_REAL_IF, fs, g["if_hz"], blocks,
                        np.arange(1, 33, dtype=np.int32), bins, device_ptr=raw.data_ptr())
    x = oracle_mod.ingest(raw.cpu().numpy(), abi.FMT_INT8_REAL_IF, fs, g["if_hz"])
    absent = next(p for p in range(1, 33) if p not in set(int(q) for q in prns_sv))
    for sv_i, p in ((0, int(prns_sv[0])), (1, int(prns_sv[1])), (None, absent)):
        k = int(np.argmin(np.abs(bins - svs[sv_i].doppler_hz))) if sv_i is not None else 20
        sel = sorted({max(0, min(bins.size - 1, k + o)) for o in (-1, 0, 1)})
        want = oracle_mod.ref_pcs_plane(x, blocks, p, fs, bins[sel])[:, ::8]
        err = np.abs(plane[p - 1][sel] - want).max() / want.max()
        assert err < 1e-5, (p, err)
