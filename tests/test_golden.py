"""Golden fixtures generated from the reference itself
(tests/golden/make_golden.py -> golden_r1.npz).  The CPU tests pin the
oracle to them (no reference build needed, so they also run on the GPU
box); the gpu tests check libl1rxg against the same reference outputs."""
import os

import numpy as np
import pytest

from paper_1907_00463_b200 import abi

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_r1.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def _cases(g):
    off = 0
    for k in range(len(g["corr_n"])):
        n = int(g["corr_n"][k])
        iq8 = g["corr_iq8"][off:off + 2 * n].reshape(n, 2).astype(np.float64)
        off += 2 * n
        x = (iq8[:, 0] + 1j * iq8[:, 1]) / 128.0
        yield k, float(g["corr_fs"][k]), x, abi.Nco(*g["corr_nco_in"][k]), int(g["corr_prn"][k]), \
            float(g["corr_spacing"][k])


def test_codes(g, oracle_mod):
    for p in range(1, 33):
        assert np.array_equal(oracle_mod.ca_code(p), g["codes"][p - 1])


def test_oracle_correlator_vs_reference_fixture(g, oracle_mod):
    for k, fs, x, nco, prn, sp in _cases(g):
        o, _, adv = oracle_mod.correlate(x, nco, prn, abi.Taps.epl(sp), fs)
        want = g["corr_sums_scalar"][k]
        got = np.array(o.as_tuple())
        assert np.abs(got - want).max() <= 1e-12 * max(np.abs(want[:6]).max(), 1e-9)
        assert (adv.code_phase_chips, adv.carrier_phase_rad, adv.chi_chips) == \
            tuple(g["corr_nco_out"][k][[0, 3, 4]])
        # the reference's own batched kernel agrees with its scalar one to 1e-6
        b = g["corr_sums_batched"][k]
        assert np.abs(b - want).max() <= 1e-6 * max(np.abs(want[:6]).max(), 1e-9)


def test_oracle_ingest_vs_reference_fixture(g, oracle_mod):
    for tag in ("if4", "gn3s"):
        fs, ifz = g[f"ingest_{tag}_rate"]
        out = oracle_mod.ingest(g[f"ingest_{tag}_raw"].view(np.uint8), abi.FMT_INT8_REAL_IF, fs, ifz)
        assert np.abs(out - g[f"ingest_{tag}_out"]).max() < 1e-12


def test_oracle_loop_vs_reference_fixture(g, oracle_mod):
    fs = float(g["loop_fs"][0])
    q = g["loop_iq8"].reshape(-1, 2).astype(np.float64)
    x = (q[:, 0] + 1j * q[:, 1]) / 128.0
    init = abi.Channel.from_buffer_copy(g["loop_init"].tobytes())
    ref = g["loop_records"]
    _, done, recs, _ = oracle_mod.track_run([init], [0], [x], 2048, abi.TrackingCfg.default(),
                                            abi.Taps.epl(0.5), fs, 400)
    got = recs[0][: done[0]]
    assert len(got) == len(ref)
    for f in ("ip", "qp", "ie", "qe", "il", "ql", "carrier_doppler_hz", "code_freq_hz", "cn0_dbhz",
              "carrier_lock_ratio", "pll_integrator", "dll_integrator"):
        scale = max(np.abs(ref[f]).max(), 1.0)
        assert np.abs(got[f] - ref[f]).max() <= 1e-9 * scale, f
    assert np.array_equal(got["chi_chips"], ref["chi_chips"])
    assert np.array_equal(got["state"], ref["state"])


@pytest.mark.gpu
def test_gpu_correlator_vs_reference_fixture(g, ctx):
    """GPU per-call path vs the reference's correlate_epoch_scalar outputs."""
    for k, fs, x, nco, prn, sp in _cases(g):
        st = abi.Nco.from_buffer_copy(nco)
        o = ctx.correlate_epoch(x, st, prn, sp, fs)
        want = g["corr_sums_scalar"][k]
        got = np.array(o.as_tuple())
        assert np.abs(got - want).max() <= 1e-5 * max(np.abs(want[:6]).max(), 1e-9), k
        assert (st.code_phase_chips, st.carrier_phase_rad, st.chi_chips) == \
            tuple(g["corr_nco_out"][k][[0, 3, 4]])


@pytest.mark.gpu
def test_gpu_ingest_vs_reference_fixture(g, ctx):
    from paper_1907_00463_b200.tracking import Tracker
    for tag in ("if4", "gn3s"):
        fs, ifz = g[f"ingest_{tag}_rate"]
        raw = g[f"ingest_{tag}_raw"]
        trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, fs, ifz, [], ring_samples=1 << 16)
        trk.push(0, raw[:2500])
        trk.push(0, raw[2500:])
        got = trk.read_samples(0, 0, raw.size)
        assert np.abs(got - g[f"ingest_{tag}_out"]).max() < 2e-6


@pytest.mark.gpu
def test_gpu_loop_vs_reference_fixture(g, ctx, oracle_mod):
    """Closed loop on the GPU from the reference's own hand-off state; per-
    epoch replay parity plus whole-run agreement with the reference records."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from helpers import replay_check
    from paper_1907_00463_b200.tracking import Tracker
    fs = float(g["loop_fs"][0])
    init = abi.Channel.from_buffer_copy(g["loop_init"].tobytes())
    trk = Tracker(ctx, abi.FMT_INT8_IQ, fs, 0.0, [init], ring_samples=1 << 20, max_records=256)
    trk.push(0, g["loop_iq8"])
    trk.run()
    recs = trk.records(0)
    ref = g["loop_records"]
    assert len(recs) == len(ref)
    q = g["loop_iq8"].reshape(-1, 2).astype(np.float64)
    x = (q[:, 0] + 1j * q[:, 1]) / 128.0
    replay_check(oracle_mod, init, recs, x, 2048, abi.TrackingCfg.default(), abi.Taps.epl(0.5), fs)
    d = np.abs(recs["carrier_doppler_hz"] - ref["carrier_doppler_hz"]).max()
    assert d < 1e-3, d
    assert np.abs(recs["chi_chips"] - ref["chi_chips"]).max() < 1e-6
