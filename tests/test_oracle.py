"""Pins the CPU oracle (oracle/l1rx_oracle.c) before any GPU result is
trusted: against the reference itself (oracle/_ref, the unmodified l1rx
headers compiled in place) and against the reference's own known-answer
tests restated (test_cacode.cpp, test_tracking.cpp, test_samples.cpp)."""
import math

import numpy as np
import pytest

from paper_1907_00463_b200 import abi


@pytest.fixture(scope="module")
def orc(oracle_mod):
    return oracle_mod


def need_ref(orc):
    if not orc.ref_available():
        pytest.skip("reference library not built (no /root/reference here)")


# ---- C/A codes (test_cacode.cpp) ----------------------------------------

def test_prn1_starts_with_octal_1440(orc):
    c = orc.ca_code(1)
    assert list(c[:10]) == [1 - 2 * b for b in (1, 1, 0, 0, 1, 0, 0, 0, 0, 0)]


def test_codes_match_delay_based_generator(orc):
    """test_cacode.cpp:18-45 independent generator (per-PRN G2 delays)."""
    g2_delay = [0, 5, 6, 7, 8, 17, 18, 139, 140, 141, 251, 252, 254, 255, 256, 257, 258, 469, 470,
                471, 472, 473, 474, 509, 512, 513, 514, 515, 516, 859, 860, 861, 862]
    r1, r2 = [-1] * 10, [-1] * 10
    g1, g2 = [], []
    for _ in range(1023):
        g1.append(r1[9])
        g2.append(r2[9])
        s1 = r1[2] * r1[9]
        s2 = r2[1] * r2[2] * r2[5] * r2[7] * r2[8] * r2[9]
        r1 = [s1] + r1[:9]
        r2 = [s2] + r2[:9]
    for prn in range(1, 33):
        d = g2_delay[prn]
        want = [g1[i] * g2[(i - d + 1023) % 1023] for i in range(1023)]
        assert list(orc.ca_code(prn)) == want, prn


def test_code_balance_and_correlation(orc):
    codes = {p: orc.ca_code(p).astype(np.int64) for p in range(1, 33)}
    for p, c in codes.items():
        assert sorted([(c > 0).sum(), (c < 0).sum()]) == [511, 512]
        ac = np.array([int(np.dot(c, np.roll(c, -lag))) for lag in range(1023)])
        assert ac[0] == 1023 and set(ac[1:]) <= {-65, -1, 63}
    for a, b in [(1, 2), (7, 13), (21, 32)]:
        cc = {int(np.dot(codes[a], np.roll(codes[b], -lag))) for lag in range(1023)}
        assert cc <= {-65, -1, 63}


def test_prn_out_of_range(orc):
    with pytest.raises(IndexError):
        orc.ca_code(0)
    with pytest.raises(IndexError):
        orc.ca_code(33)


def test_codes_equal_reference(orc):
    need_ref(orc)
    for p in range(1, 33):
        assert np.array_equal(orc.ca_code(p), orc.ca_code(p, "ref"))


# ---- ingest (samples.hpp) -------------------------------------------------

def test_int_decode_known_values(orc):
    """test_samples.cpp:42-67."""
    x = orc.ingest(np.array([100, 256 - 50, 0, 127], np.uint8), abi.FMT_INT8_IQ, 5e6)
    assert x[0] == complex(100 / 128.0, -50 / 128.0) and x[1] == complex(0.0, 127 / 128.0)
    y = orc.ingest(np.array([0x02, 0x01, 0xFE, 0xFF], np.uint8), abi.FMT_INT16_IQ, 5e6)
    assert y[0] == complex(258 / 32768.0, -2 / 32768.0)


def test_halfband_taps(orc):
    h = np.zeros(23)
    orc.port().orc_halfband_taps(orc.dptr(h))
    assert abs(h.sum() - 1.0) < 1e-15 and h[11] == pytest.approx(0.501105, abs=1e-6)
    assert np.abs(h - h[::-1]).max() < 1e-15
    assert np.abs(h[1::2][:5]).max() < 1e-16 + 2e-17  # even k (odd n) taps ~ 0


@pytest.mark.parametrize("fmt,fs,ifz", [(abi.FMT_INT8_REAL_IF, 16.368e6, 4.092e6),
                                        (abi.FMT_INT8_REAL_IF, 16.3676e6, 4.1304e6),
                                        (abi.FMT_INT8_IQ, 5e6, 0.0),
                                        (abi.FMT_INT16_IQ, 65.472e6, 0.0)])
def test_ingest_equals_sample_source(orc, fmt, fs, ifz):
    need_ref(orc)
    rng = np.random.default_rng(5)
    raw = rng.integers(0, 256, 60_000).astype(np.uint8)
    a = orc.ingest(raw, fmt, fs, ifz)
    b = orc.ref_ingest(raw, fmt, fs, ifz)
    assert a.size == b.size
    assert np.abs(a - b).max() < 1e-12


def test_real_if_tone_lands_at_baseband(orc):
    """test_samples.cpp:174-227 (numpy FFT instead of FFTW)."""
    fs, ifz, off, n = 16.3676e6, 4.1304e6, 50e3, 16384
    t = np.arange(n) / fs
    raw = np.round(100.0 * np.cos(2 * np.pi * (ifz + off) * t)).astype(np.int8)
    x = orc.ingest(raw.view(np.uint8), abi.FMT_INT8_REAL_IF, fs, ifz)
    spec = np.fft.fft(x)
    peak = int(np.argmax(np.abs(spec)))
    f = peak * fs / n
    f = f - fs if f > fs / 2 else f
    assert abs(f - off) <= fs / n
    img = int(round((-2 * ifz - off) / (fs / n) + n)) % n
    assert np.abs(spec[img]) < np.abs(spec[peak]) / 10


# ---- correlator (tracking.hpp:226-429) --------------------------------------

def _naive(view, nco, code, spacing, fs):
    """test_tracking.cpp:51-77 plain-loop oracle."""
    w = 2 * math.pi * nco.carrier_doppler_hz / fs
    cps = nco.code_freq_hz / fs
    i = np.arange(view.size)
    th = nco.carrier_phase_rad + w * i
    wiped = view * (np.cos(th) - 1j * np.sin(th))
    ph = nco.code_phase_chips + i * cps + 2046.0

    def chip(p):
        return code[np.fmod(np.floor(p), 1023.0).astype(np.int64)].astype(np.float64)
    e, p, l = chip(ph + spacing / 2), chip(ph), chip(ph - spacing / 2)
    return np.array([np.sum(wiped.real * e), np.sum(wiped.imag * e), np.sum(wiped.real * p),
                     np.sum(wiped.imag * p), np.sum(wiped.real * l), np.sum(wiped.imag * l)])


def test_correlator_matches_naive_oracle(orc):
    rng = np.random.default_rng(11)
    fs = 5e6
    code = orc.ca_code(7)
    for _ in range(20):
        view = rng.uniform(-1, 1, 5000) + 1j * rng.uniform(-1, 1, 5000)
        nco = abi.Nco(rng.uniform(0, 1023), 1.023e6 + rng.uniform(-3, 3), rng.uniform(-5000, 5000),
                      rng.uniform(0, 2 * math.pi), 0.0)
        o, _, _ = orc.correlate(view, nco, 7, abi.Taps.epl(0.5), fs)
        want = _naive(view, nco, code, 0.5, fs)
        got = np.array(o.as_tuple()[:6])
        scale = max(abs(want[2]), abs(want[3]), abs(want[0]), 1e-12)
        assert np.abs(got - want).max() < 1e-9 * scale


@pytest.mark.parametrize("fs", [5e6, 16.368e6, 65.472e6, 2.048e6])
@pytest.mark.parametrize("kernel", [0, 1])
def test_correlator_equals_reference(orc, fs, kernel):
    """3-tap restatement vs the reference's scalar (bit-identical NCO advance
    and chip decisions, sums to fp64 rounding) and batched kernels."""
    need_ref(orc)
    rng = np.random.default_rng(int(fs) % 1009 + kernel)
    n = int(round(fs / 1000))
    for trial in range(12):
        view = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        if trial % 3 == 0:
            nco = abi.Nco(float(rng.integers(0, 16368)) / 16.0, 1.023e6, 0.0, 0.0, 0.0)
        else:
            nco = abi.Nco(rng.uniform(0, 1023), 1.023e6 + rng.uniform(-3, 3),
                          rng.uniform(-5000, 5000), rng.uniform(0, 2 * math.pi), 0.0)
        prn = int(rng.integers(1, 33))
        a, sa = orc.ref_correlate(view, nco, prn, 0.5, fs, kernel=kernel)
        b, _, sb = orc.correlate(view, nco, prn, abi.Taps.epl(0.5), fs)
        at, bt = np.array(a.as_tuple()), np.array(b.as_tuple())
        tol = 1e-12 if kernel == 0 else 1e-6  # batched = scalar to 1e-6 (test_tracking.cpp:166-204)
        assert np.abs(at - bt).max() <= tol * max(np.abs(at[:6]).max(), 1e-9)
        assert (sa.code_phase_chips, sa.carrier_phase_rad, sa.chi_chips) == \
            (sb.code_phase_chips, sb.carrier_phase_rad, sb.chi_chips)


def test_ktap_three_tap_instance_is_reference(orc):
    """The K-tap restatement (builder extension) with offsets (+s/2,0,-s/2)
    is the reference expression: tap sums identical to the E/P/L path."""
    rng = np.random.default_rng(21)
    fs = 16.368e6
    view = rng.uniform(-1, 1, 16368) + 1j * rng.uniform(-1, 1, 16368)
    nco = abi.Nco(100.2, 1.023e6 + 0.3, 321.0, 0.4, 0.0)
    o, sums, _ = orc.correlate(view, nco, 4, abi.Taps.epl(0.5), fs)
    t5 = abi.Taps.make([0.5, 0.25, 0.0, -0.25, -0.5], early=1, prompt=2, late=3)
    o5, s5, _ = orc.correlate(view, nco, 4, t5, fs)
    assert np.array_equal(s5[2:8], sums)
    assert o5.ip_h1 == o.ip_h1


def test_empty_view_is_an_error(orc):
    with pytest.raises(ValueError):
        orc.correlate(np.zeros(0, np.complex128), abi.Nco(0, 1.023e6, 0, 0, 0), 7,
                      abi.Taps.epl(0.5), 5e6)


# ---- loop (tracking.hpp:65-147, 459-650) -----------------------------------

def test_discriminators_and_filter(orc):
    """test_tracking.cpp:250-320 known answers."""
    P = orc.port()
    c = abi.Corr()
    c.ie, c.il = 0.5, 0.5
    assert P.orc_dll_discriminator(c) == 0.0
    c = abi.Corr()
    c.ie = 1.0
    assert P.orc_dll_discriminator(c) == pytest.approx(0.5)
    c = abi.Corr()
    c.ie, c.il = 0.6, 1.0
    assert P.orc_dll_discriminator(c) == pytest.approx(-0.125)
    assert P.orc_dll_discriminator(abi.Corr()) == 0.0
    assert P.orc_pll_discriminator(1, 0) == 0.0
    assert P.orc_pll_discriminator(1, 1) == pytest.approx(math.pi / 4)
    assert P.orc_pll_discriminator(-1, 1) == pytest.approx(-math.pi / 4)
    assert P.orc_pll_discriminator(0, -3) == pytest.approx(-math.pi / 2)
    assert P.orc_fll_discriminator(1, 0, 1, 0, 1e-3) == 0.0
    assert P.orc_fll_discriminator(1, 0, 0, 1, 1e-3) == pytest.approx(250.0)
    w = 2 * math.pi * 100.0 * 1e-3
    assert P.orc_fll_discriminator(1, 0, math.cos(w), math.sin(w), 1e-3) == pytest.approx(100.0, rel=1e-6)
    assert P.orc_carrier_aid(0.0, 0.0) == 1.023e6
    assert P.orc_carrier_aid(1575.42, 0.0) == pytest.approx(1.023e6 + 1.023, rel=1e-12)
    import ctypes as C
    i, p, pr = C.c_double(0), C.c_double(0), C.c_int32(0)
    for _ in range(100):
        assert P.orc_loop_filter_update(C.byref(i), C.byref(p), C.byref(pr), 0.0, 25.0, 0.707, 1e-3) == 0.0


def test_discriminators_equal_reference(orc):
    need_ref(orc)
    P, R = orc.port(), orc.ref()
    rng = np.random.default_rng(9)
    import ctypes as C
    for _ in range(200):
        v = rng.normal(size=6)
        c = abi.Corr()
        c.ie, c.qe, c.ip, c.qp, c.il, c.ql = v
        # the reference build contracts a*a+b*b etc. into FMAs; the
        # restatement agrees to a few ulp (carrier aiding, which feeds the
        # code NCO, is matched bit for bit)
        assert P.orc_dll_discriminator(c) == pytest.approx(R.ref_dll_discriminator(c), rel=1e-13, abs=1e-15)
        assert P.orc_pll_discriminator(v[2], v[3]) == pytest.approx(R.ref_pll_discriminator(v[2], v[3]), rel=1e-13)
        a = list(rng.normal(size=4)) + [1e-3]
        assert P.orc_fll_discriminator(*a) == pytest.approx(R.ref_fll_discriminator(*a), rel=1e-12, abs=1e-9)
        assert P.orc_fll_discriminator_di(*a) == pytest.approx(R.ref_fll_discriminator_di(*a), rel=1e-12, abs=1e-9)
        assert P.orc_carrier_aid(v[0] * 3000, v[1]) == R.ref_carrier_aid(v[0] * 3000, v[1])
        i1, p1, q1 = C.c_double(v[4]), C.c_double(v[5]), C.c_int32(1)
        i2, p2, q2 = C.c_double(v[4]), C.c_double(v[5]), C.c_int(1)
        assert P.orc_loop_filter_update(C.byref(i1), C.byref(p1), C.byref(q1), v[0], 25.0, 0.707, 1e-3) == \
            pytest.approx(R.ref_loop_filter_update(C.byref(i2), C.byref(p2), C.byref(q2), v[0], 25.0, 0.707, 1e-3), rel=1e-13)


def test_init_channel_equals_reference(orc):
    need_ref(orc)
    from paper_1907_00463_b200.tracking import init_channel_from_acquisition
    rng = np.random.default_rng(4)
    for _ in range(50):
        # 2.0465 MHz: samples per ms 2046.5 -- llround rounds the half away from zero
        fs = float(rng.choice([2.048e6, 2.0465e6, 5e6, 16.368e6, 65.472e6]))
        args = (int(rng.integers(1, 33)), rng.uniform(-5000, 5000), int(rng.integers(0, 10**6)),
                int(rng.integers(0, 70000)), int(rng.integers(0, 2 * 10**6)), fs)
        a = orc.init_channel(*args, which="ref")
        b = orc.init_channel(*args, which="port")
        c = init_channel_from_acquisition(*args)
        assert bytes(a) == bytes(b) == bytes(c)


@pytest.mark.parametrize("window_ms", [20, 100])
def test_closed_loop_equals_reference(orc, window_ms):
    """track_epoch restatement vs the reference over a 1.5 s closed loop
    (test_tracking.cpp:403-417 scenario); at cn0_window_ms = 100 the
    restatement carries the window as running sums (longer than the POD's
    64-entry arrays, l1rxg.h) and must still equal the reference's vectors."""
    need_ref(orc)
    fs = 2.048e6
    sig = orc.ref_sim_baseband([dict(prn=7, cn0=45, doppler=320.0, delay_chips=100.25)], 1.5, fs,
                               True, 77)
    b = int(round(100.25 / 1.023e6 * fs))
    ch = orc.init_channel(7, 0.0, 0, b - 1, 0, fs, "ref")
    cfg = abi.TrackingCfg.default()
    cfg.cn0_window_ms = window_ms
    _, r = orc.ref_track_buffer(ch, sig, 2048, cfg, fs, kernel=0)
    _, done, p, _ = orc.track_run([ch], [0], [sig], 2048, cfg, abi.Taps.epl(0.5), fs, 2000)
    p = p[0][: done[0]]
    assert len(p) == len(r) >= 1400
    for f in ("ip", "qp", "ie", "ql", "carrier_doppler_hz", "cn0_dbhz", "carrier_lock_ratio"):
        scale = max(np.abs(r[f]).max(), 1.0)
        assert np.abs(p[f] - r[f]).max() <= 1e-9 * scale, f
    assert np.array_equal(p["chi_chips"], r["chi_chips"])
    assert r[1000]["carrier_lock_ratio"] > 0.9
    assert abs(r[1000]["carrier_doppler_hz"] - 320.0) < 5.0


def test_quality_metrics_clean_prompts(orc):
    """test_tracking.cpp:341-359."""
    P = orc.port()
    cfg = abi.TrackingCfg.default()
    import ctypes as C
    for ip, qp, lo, cn0 in ((2.0, 0.0, 0.999, 65.0), (0.0, 2.0, None, None)):
        ch = abi.Channel()
        ch.state = abi.TRACKING
        o = abi.Corr()
        o.ip, o.qp = ip, qp
        for _ in range(200):
            P.orc_update_quality_metrics(C.byref(ch), C.byref(o), C.byref(cfg))
        if lo is not None:
            assert ch.carrier_lock_ratio > lo and ch.cn0_dbhz == pytest.approx(cn0)
        else:
            assert ch.carrier_lock_ratio < -0.999


def test_silence_drops_channel(orc):
    """test_tracking.cpp:431-447 on the oracle."""
    fs = 2.048e6
    ch = orc.init_channel(7, 0.0, 0, 0, 0, fs)
    sig = np.zeros(2048 * 80, np.complex128)
    out, done, _, _ = orc.track_run([ch], [0], [sig], 2048, abi.TrackingCfg.default(),
                                    abi.Taps.epl(0.5), fs, 80)
    assert out[0].state == abi.IDLE and done[0] == 51


def test_search_grid_recovers_delay_and_doppler(orc):
    """acquire_pcs semantics (acquisition.hpp:189-222) on a small grid:
    the peak sits at the true code delay and Doppler bin (the property
    test_acquisition.cpp:145-160 pins)."""
    fs = 2.046e6  # 2 samples/chip keeps the direct evaluation quick
    N = 2046
    from paper_1907_00463_b200 import simsource as ss
    sv = ss.Sv(prn=13, cn0_dbhz=50.0, doppler_hz=1500.0, delay_chips=200.0)
    raw = ss.synth(4, fs, [sv], fmt="int16_iq", seed=3).numpy()
    x = orc.ingest(raw, abi.FMT_INT16_IQ, fs)
    bins = np.arange(-5000.0, 5000.1, 500.0)
    plane = orc.search_grid(x, N, 4, 13, fs, bins, 1, N)
    b, d = np.unravel_index(np.argmax(plane), plane.shape)
    assert bins[b] == 1500.0
    assert abs(d - 400) <= 1
