"""GPU correlator (K2) parity against the oracle, through the C ABI.

Bars: chip decisions bit-exact; sums within 1e-5 x max of the
E/P/L sums (the reference's own normalisation, test_tracking.cpp:189-197);
NCO state advance bit-exact (the reference checks 1e-9, :199-202)."""
import math

import numpy as np
import pytest

from paper_1907_00463_b200 import abi

pytestmark = pytest.mark.gpu

RATES = [16.368e6, 5e6, 65.472e6, 2.048e6]
TAPSETS = {
    "epl": abi.Taps.epl(0.5),
    "epl_narrow": abi.Taps.epl(0.2),
    # spoofing monitor: 11 taps on a 0.1-chip grid + loop E/L at +/-0.25
    "monitor13": abi.Taps.make([round(-0.5 + 0.1 * k, 10) for k in range(11)] + [0.25, -0.25],
                               early=11, prompt=5, late=12, n_counted=11),
    # wideband batch: 7 taps on a 0.25-chip grid, E/L = +/-0.25
    "wide7": abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2),
}


def _states(rng, nj, fs, exact_ties=False):
    states, prns = [], []
    for j in range(nj):
        if exact_ties and j % 2 == 0:
            # commensurate code rate and grid-aligned phase: chip boundaries
            # land exactly on samples (the tie regime, proj/README.md:127-131)
            cf = 1.023e6
            cp = float(rng.integers(0, 1023 * 16)) / 16.0
        else:
            cf = 1.023e6 + rng.uniform(-3, 3)
            cp = rng.uniform(0, 1023)
        states.append(abi.Nco(cp, cf, 0.0, 0.0, rng.uniform(0, 1e6)))
        prns.append(int(rng.integers(1, 33)))
    return states, prns


@pytest.mark.parametrize("fs", RATES)
@pytest.mark.parametrize("tapset", list(TAPSETS))
def test_chip_decisions_bit_exact(ctx, oracle_mod, fs, tapset):
    """Zero Doppler/phase and k/128-valued inputs make every fp32 operation
    of the GPU path exact, so any chip-decision difference from the
    reference expression would show up as an exact mismatch."""
    taps = TAPSETS[tapset]
    rng = np.random.default_rng(int(fs) % 1000 + len(tapset))
    n = int(round(fs / 1000))
    nj = 24
    iq = (rng.integers(-7, 8, (nj, n)) + 1j * rng.integers(-7, 8, (nj, n))) / 128.0
    states, prns = _states(rng, nj, fs, exact_ties=True)
    st_gpu = [abi.Nco.from_buffer_copy(s) for s in states]
    sums, corr = ctx.correlate_batch(iq, st_gpu, prns, taps, fs)
    for j in range(nj):
        o, want, adv = oracle_mod.correlate(iq[j], states[j], prns[j], taps, fs)
        assert np.array_equal(sums[j], want), f"job {j}: tap sums differ {sums[j] - want}"
        assert corr[j].ip_h1 == o.ip_h1 and corr[j].qp_h1 == o.qp_h1
        assert (st_gpu[j].code_phase_chips, st_gpu[j].carrier_phase_rad, st_gpu[j].chi_chips) == \
            (adv.code_phase_chips, adv.carrier_phase_rad, adv.chi_chips)


@pytest.mark.parametrize("fs", RATES)
@pytest.mark.parametrize("tapset", list(TAPSETS))
def test_random_epochs_within_tolerance(ctx, oracle_mod, fs, tapset):
    taps = TAPSETS[tapset]
    rng = np.random.default_rng(7 + int(fs) % 997)
    n = int(round(fs / 1000))
    nj = 40
    iq = rng.uniform(-1, 1, (nj, n)) + 1j * rng.uniform(-1, 1, (nj, n))
    states = []
    prns = []
    for _ in range(nj):
        states.append(abi.Nco(rng.uniform(0, 1023), 1.023e6 + rng.uniform(-3, 3),
                              rng.uniform(-5000, 5000), rng.uniform(0, 2 * math.pi), 0.0))
        prns.append(int(rng.integers(1, 33)))
    st_gpu = [abi.Nco.from_buffer_copy(s) for s in states]
    sums, corr = ctx.correlate_batch(iq, st_gpu, prns, taps, fs)
    worst = 0.0
    for j in range(nj):
        o, want, adv = oracle_mod.correlate(iq[j], states[j], prns[j], taps, fs)
        scale = max(np.abs(want).max(), 1e-9)
        err = np.abs(sums[j] - want).max() / scale
        h = np.array([corr[j].ip_h1, corr[j].qp_h1, corr[j].ip_h2, corr[j].qp_h2])
        hw = np.array([o.ip_h1, o.qp_h1, o.ip_h2, o.qp_h2])
        err = max(err, np.abs(h - hw).max() / scale)
        worst = max(worst, err)
        assert err <= 1e-5, f"job {j}: rel err {err:.3g}"
        assert st_gpu[j].code_phase_chips == adv.code_phase_chips
        assert st_gpu[j].carrier_phase_rad == adv.carrier_phase_rad
        assert st_gpu[j].chi_chips == adv.chi_chips
    print(f"{tapset} @ {fs/1e6} MHz worst rel err {worst:.3g}")


def test_per_call_path_matches_reference_scalar(ctx, oracle_mod):
    """l1rxg_correlate_epoch vs the reference's own correlate_epoch_scalar
    (oracle/_ref), 200 random epochs at 5 MHz as in test_tracking.cpp:166-204
    (batched = scalar to 1e-6 there; the GPU bar is 1e-5)."""
    if not oracle_mod.ref_available():
        pytest.skip("reference library not built")
    rng = np.random.default_rng(12)
    fs = 5e6
    for trial in range(200):
        view = rng.uniform(-1, 1, 5000) + 1j * rng.uniform(-1, 1, 5000)
        nco = abi.Nco(rng.uniform(0, 1023), 1.023e6 + rng.uniform(-3, 3),
                      rng.uniform(-5000, 5000), rng.uniform(0, 2 * math.pi), 0.0)
        prn = int(rng.integers(1, 33))
        a, sa = oracle_mod.ref_correlate(view, nco, prn, 0.5, fs, kernel=0)
        ch = abi.Nco.from_buffer_copy(nco)
        b = ctx.correlate_epoch(view, ch, prn, 0.5, fs)
        at, bt = np.array(a.as_tuple()), np.array(b.as_tuple())
        scale = max(np.abs(at[:6]).max(), 1e-9)
        assert np.abs(at - bt).max() <= 1e-5 * scale
        assert ch.code_phase_chips == sa.code_phase_chips
        assert ch.carrier_phase_rad == sa.carrier_phase_rad
        assert ch.chi_chips == sa.chi_chips
        assert b.n_samples == 5000


def test_errors_match_reference(ctx):
    """test_tracking.cpp:238-248 (empty view) and cacode.hpp:38-39 (PRN)."""
    ch = abi.Nco(0.0, 1.023e6, 0.0, 0.0, 0.0)
    with pytest.raises(ValueError, match="empty epoch view"):
        ctx.correlate_epoch(np.zeros(0, np.complex128), ch, 7, 0.5, 5e6)
    with pytest.raises(IndexError):
        ctx.correlate_epoch(np.zeros(5000, np.complex128), ch, 33, 0.5, 5e6)
    with pytest.raises(ValueError):
        ctx.correlate_batch(np.zeros((1, 100), np.complex128), [ch], [1],
                            abi.Taps.make([0.0], 0, 0, 0), 0.0)


def test_noop_kernel_advances_state(ctx):
    """correlate_epoch_noop (tracking.hpp:434-452)."""
    fs = 2.048e6
    ch = abi.Nco(5.0, 1.023e6 + 0.6, 1000.0, 0.3, 5.0)
    out = ctx.correlate_epoch(np.full(2048, 0.5 - 0.25j), ch, 7, 0.5, fs, kernel=abi.KERNEL_NOOP)
    assert out.ip == 0.0 and out.n_samples == 2048
    assert ch.chi_chips == pytest.approx(5.0 + 2048 * (1.023e6 + 0.6) / fs, abs=1e-9)


def _sim(oracle_mod, cn0, doppler, delay, fs, dur, noise, seed):
    return oracle_mod.ref_sim_baseband([dict(prn=7, cn0=cn0, doppler=doppler, delay_chips=delay)],
                                       dur, fs, noise, seed)


def test_aligned_noiseless_replica(ctx, oracle_mod):
    """test_tracking.cpp:81-95 on the GPU path (tolerances at the GPU's
    1e-5 bar instead of the fp64 kernel's 1e-9)."""
    if not oracle_mod.ref_available():
        pytest.skip("reference library not built")
    fs = 5e6
    sig = _sim(oracle_mod, 48, 0, 0, fs, 0.001, False, 1)
    ch = abi.Nco(0.0, 1.023e6, 0.0, 0.0, 0.0)
    out = ctx.correlate_epoch(sig, ch, 7, 0.5, fs)
    amp = math.sqrt(10 ** 4.8 / fs)
    assert out.ip == pytest.approx(5000.0 * amp, rel=1e-5)
    assert abs(out.qp) < 1e-5 * out.ip
    e_env, l_env = math.hypot(out.ie, out.qe), math.hypot(out.il, out.ql)
    assert e_env == pytest.approx(l_env, rel=1e-2)
    assert out.ip > e_env


def test_late_beats_early_and_dll_odd(ctx, oracle_mod):
    """test_tracking.cpp:97-128."""
    if not oracle_mod.ref_available():
        pytest.skip("reference library not built")
    fs = 5e6
    sig = _sim(oracle_mod, 48, 0, 0.1, fs, 0.001, False, 2)
    out = ctx.correlate_epoch(sig, abi.Nco(0.0, 1.023e6, 0.0, 0.0, 0.0), 7, 0.5, fs)
    assert math.hypot(out.il, out.ql) > math.hypot(out.ie, out.qe)
    for delta in (0.05, 0.2, 0.4):
        sp = _sim(oracle_mod, 48, 0, delta, fs, 0.001, False, 3)
        sm = _sim(oracle_mod, 48, 0, 1023.0 - delta, fs, 0.001, False, 3)
        op = ctx.correlate_epoch(sp, abi.Nco(0.0, 1.023e6, 0.0, 0.0, 0.0), 7, 0.5, fs)
        om = ctx.correlate_epoch(sm, abi.Nco(0.0, 1.023e6, 0.0, 0.0, 0.0), 7, 0.5, fs)
        ep = oracle_mod.port().orc_dll_discriminator(op)
        em = oracle_mod.port().orc_dll_discriminator(om)
        assert ep == pytest.approx(-em, abs=2e-3)
        assert ep < 0
