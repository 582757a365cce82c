"""Closed-loop tracking on the GPU (K1 ingest + K2 correlator + K3 loop
update on device) against the oracle, through the C ABI.

The binding parity check is per-epoch replay: every GPU
epoch is re-run by the oracle from the GPU's own pre-epoch state.  Whole-run
behaviour is checked with the reference's own closed-loop criteria
(test_tracking.cpp:403-479)."""
import math

import os

import numpy as np
import pytest

from paper_1907_00463_b200 import abi, simsource as ss
from paper_1907_00463_b200.tracking import Tracker, init_channel_from_acquisition

from helpers import replay_check

pytestmark = pytest.mark.gpu

IF_FS, IF_HZ = 16.368e6, 4.092e6


def _raw(n_ms, fs, svs, fmt, if_hz=0.0, seed=1):
    return ss.synth(n_ms, fs, svs, fmt=fmt, if_hz=if_hz, seed=seed, device="cuda").cpu().numpy()


def _init(sv, fs, dop_err=0.0, samp_err=0):
    b, d = ss.truth_channel_start(sv, fs)
    return init_channel_from_acquisition(sv.prn, d - dop_err, 0, b + samp_err, 0, fs)


def test_ingest_real_if_matches_sample_source(ctx, oracle_mod):
    """K1 vs SampleSource's mixer + half-band FIR (samples.hpp:215-253),
    pushed in uneven chunks so the carried FIR history is exercised."""
    rng = np.random.default_rng(3)
    raw = rng.integers(-128, 128, 200_003).astype(np.int8)
    trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, IF_FS, IF_HZ, [], ring_samples=1 << 20)
    pos = 0
    for step in (17, 16368, 5, 100_000, 83_613):
        trk.push(0, raw[pos:pos + step])
        pos += step
    got = trk.read_samples(0, 0, raw.size)
    want = oracle_mod.ingest(raw, abi.FMT_INT8_REAL_IF, IF_FS, IF_HZ)
    if oracle_mod.ref_available():
        ref = oracle_mod.ref_ingest(raw, abi.FMT_INT8_REAL_IF, IF_FS, IF_HZ)
        assert np.abs(ref - want).max() < 1e-12
    assert np.abs(got - want).max() < 2e-6


def test_ingest_generic_if_and_complex_formats(ctx, oracle_mod):
    rng = np.random.default_rng(4)
    # non-fs/4 IF (GN3S rates of test_samples.cpp:174-227): generic mixer path
    fs, ifz = 16.3676e6, 4.1304e6
    raw = rng.integers(-128, 128, 50_000).astype(np.int8)
    trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, fs, ifz, [], ring_samples=1 << 18)
    trk.push(0, raw[:20_000])
    trk.push(0, raw[20_000:])
    got = trk.read_samples(0, 0, raw.size)
    want = oracle_mod.ingest(raw, abi.FMT_INT8_REAL_IF, fs, ifz)
    assert np.abs(got - want).max() < 2e-6
    # int8 / int16 IQ decode is exact (samples.hpp:188-205)
    for fmt, dt in ((abi.FMT_INT8_IQ, np.int8), (abi.FMT_INT16_IQ, np.int16)):
        info = np.iinfo(dt)
        raw = rng.integers(info.min, info.max + 1, 2 * 30_001).astype(dt)
        trk = Tracker(ctx, fmt, 5e6, 0.0, [], ring_samples=1 << 17)
        trk.push(0, raw)
        got = trk.read_samples(0, 0, 30_001)
        want = oracle_mod.ingest(raw.view(np.uint8), fmt, 5e6)
        assert np.array_equal(got, want)


def test_config1_shape_replay_parity(ctx, oracle_mod):
    """Config 1 shape: PRN 1, int8 real IF at 16.368 MHz / 4.092 MHz IF,
    +1.2 kHz, 45 dB-Hz, E/P/L 0.5 chip, PLL+DLL closed, 1000 blocks."""
    fs, n = IF_FS, 16368
    sv = ss.Sv(prn=1, cn0_dbhz=45.0, doppler_hz=1200.0, delay_chips=511.3)
    raw = _raw(1000, fs, [sv], "int8_real_if", IF_HZ, seed=1)
    init = _init(sv, fs, dop_err=120.0, samp_err=-1)
    cfg, taps = abi.TrackingCfg.default(), abi.Taps.epl(0.5)
    trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, fs, IF_HZ, [init], ring_samples=1100 * n,
                  max_records=1000, cfg=cfg, taps=taps)
    trk.push(0, raw)
    trk.run()
    recs, tsums = trk.records(0, tap_sums=True)
    assert len(recs) >= 998
    x = oracle_mod.ingest(raw, abi.FMT_INT8_REAL_IF, fs, IF_HZ)
    worst = replay_check(oracle_mod, init, recs, x, n, cfg, taps, fs, tap_sums=tsums)
    print("replay worst", worst)
    # reference closed-loop criteria (test_tracking.cpp:403-417)
    last = recs[-1]
    assert last["state"] == abi.TRACKING
    assert last["carrier_lock_ratio"] > 0.9
    assert abs(last["carrier_doppler_hz"] - 1200.0) < 5.0
    assert last["cn0_dbhz"] == pytest.approx(45.0, abs=3.0)


def test_trajectory_agrees_with_reference_until_first_tie(ctx, oracle_mod):
    """Whole-run agreement with the reference's own closed loop
    (oracle/_ref: SampleSource + track_epoch) on the same bytes; reported up
    to the first chip-decision tie."""
    if not oracle_mod.ref_available():
        pytest.skip("reference library not built")
    fs, n = IF_FS, 16368
    sv = ss.Sv(prn=3, cn0_dbhz=47.0, doppler_hz=-2100.0, delay_chips=100.7)
    raw = _raw(400, fs, [sv], "int8_real_if", IF_HZ, seed=5)
    init = _init(sv, fs)
    trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, fs, IF_HZ, [init], ring_samples=500 * n,
                  max_records=400)
    trk.push(0, raw)
    trk.run()
    g = trk.records(0)
    x = oracle_mod.ref_ingest(raw, abi.FMT_INT8_REAL_IF, fs, IF_HZ)
    _, r = oracle_mod.ref_track_buffer(init, x, n, abi.TrackingCfg.default(), fs, kernel=0)
    m = min(len(g), len(r))
    assert m >= 398
    d = np.abs(g["carrier_doppler_hz"][:m] - r["carrier_doppler_hz"][:m])
    chi = np.abs(g["chi_chips"][:m] - r["chi_chips"][:m])
    print("max |dDoppler| %.3g Hz, max |dchi| %.3g chips over %d epochs" % (d.max(), chi.max(), m))
    assert d.max() < 0.05 and chi.max() < 1e-3


@pytest.mark.parametrize("cta_mode", [abi.CTA_AUTO, abi.CTA_SINGLE, abi.CTA_THROUGHPUT])
def test_twelve_channel_shared_stream(ctx, oracle_mod, cta_mode):
    """Config 2 shape (scaled to 300 blocks): 12 channels, PRNs 1-12, one
    shared int8 real-IF stream, replay parity for every channel -- with each
    channel's epoch split over a cluster (auto), one CTA per channel, and the
    narrow four-per-SM throughput CTAs (several tiles per epoch)."""
    fs, n = IF_FS, 16368
    rng = np.random.default_rng(2)
    svs = [ss.Sv(prn=p, cn0_dbhz=rng.uniform(35, 50), doppler_hz=rng.uniform(-5000, 5000),
                 delay_chips=rng.uniform(0, 1023)) for p in range(1, 13)]
    raw = _raw(300, fs, svs, "int8_real_if", IF_HZ, seed=2)
    inits = [_init(sv, fs) for sv in svs]
    cfg, taps = abi.TrackingCfg.default(), abi.Taps.epl(0.5)
    trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, fs, IF_HZ, inits, ring_samples=400 * n,
                  max_records=300, cta_mode=cta_mode)
    for c0 in range(0, raw.size, 37 * n):  # chunked pushes + runs
        trk.push(0, raw[c0:c0 + 37 * n])
        trk.run()
    x = oracle_mod.ingest(raw, abi.FMT_INT8_REAL_IF, fs, IF_HZ)
    counts = trk.epoch_counts()
    for c in range(12):
        recs = trk.records(c)
        assert len(recs) == counts[c] >= 297
        replay_check(oracle_mod, inits[c], recs, x, n, cfg, taps, fs)


@pytest.mark.parametrize("chunk_blocks", [13, 7])
def test_real_if_ring_wraps(ctx, oracle_mod, chunk_blocks):
    """Real-IF stream through a ring of 40 blocks that wraps many times
    (chunked pushes + runs over 300 blocks): windows that straddle the ring's
    end, and FIR histories that reach back across it (carried by the ingest
    pass; in the raw byte ring of L1RXG_OVL_RAWIF=1 the front pad mirrors
    the tail), give the same epochs as the oracle's
    SampleSource on the whole stream; read_samples returns its baseband."""
    fs, n = IF_FS, 16368
    svs = [ss.Sv(prn=7, cn0_dbhz=46.0, doppler_hz=-1850.0, delay_chips=77.3),
           ss.Sv(prn=19, cn0_dbhz=41.0, doppler_hz=3300.0, delay_chips=903.6)]
    raw = _raw(300, fs, svs, "int8_real_if", IF_HZ, seed=17)
    inits = [_init(sv, fs) for sv in svs]
    cfg, taps = abi.TrackingCfg.default(), abi.Taps.epl(0.5)
    trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, fs, IF_HZ, inits, ring_samples=40 * n + 5,
                  max_records=300)
    x = oracle_mod.ingest(raw, abi.FMT_INT8_REAL_IF, fs, IF_HZ)
    for c0 in range(0, raw.size, chunk_blocks * n + 3):
        c1 = min(raw.size, c0 + chunk_blocks * n + 3)
        trk.push(0, raw[c0:c1])
        trk.run()
        k0 = max(0, c1 - 2 * n)
        got = trk.read_samples(0, k0, c1 - k0)
        assert np.abs(got - x[k0:c1]).max() < 2e-6
    counts = trk.epoch_counts()
    for c in range(2):
        recs = trk.records(c)
        assert len(recs) == counts[c] >= 297
        replay_check(oracle_mod, inits[c], recs, x, n, cfg, taps, fs)


@pytest.mark.parametrize("shape", ["monitor", "wideband"])
def test_multitap_replay_parity(ctx, oracle_mod, shape):
    """Configs 3 and 4 shapes (scaled): 11 taps at 0.1 chip (+2 loop taps)
    on complex int16 at 16.368 MHz; 7 taps at 0.25 chip at 65.472 MHz."""
    if shape == "monitor":
        fs = 16.368e6
        taps = abi.Taps.make([round(-0.5 + 0.1 * k, 10) for k in range(11)] + [0.25, -0.25],
                             early=11, prompt=5, late=12, n_counted=11)
        svs = [ss.Sv(prn=5, cn0_dbhz=46.0, doppler_hz=800.0, delay_chips=300.0),
               ss.Sv(prn=5, cn0_dbhz=49.0, doppler_hz=800.0, delay_chips=300.4)]
        ms = 120
    else:
        fs = 65.472e6
        taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
        svs = [ss.Sv(prn=9, cn0_dbhz=44.0, doppler_hz=-3300.0, delay_chips=12.5)]
        ms = 60
    n = int(round(fs / 1000))
    raw = _raw(ms, fs, svs, "int16_iq", seed=11)
    init = _init(svs[0], fs)
    cfg = abi.TrackingCfg.default()
    trk = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, [init], ring_samples=(ms + 8) * n,
                  max_records=ms, taps=taps, cfg=cfg)
    trk.push(0, raw.view(np.int16))
    trk.run()
    recs, tsums = trk.records(0, tap_sums=True)
    x = oracle_mod.ingest(raw, abi.FMT_INT16_IQ, fs)
    replay_check(oracle_mod, init, recs, x, n, cfg, taps, fs, tap_sums=tsums)


def test_silence_drops_to_idle(ctx):
    """test_tracking.cpp:431-447: zero input -> Idle after lock_fail_limit+1."""
    fs = 2.048e6
    init = init_channel_from_acquisition(7, 0.0, 0, 0, 0, fs)
    trk = Tracker(ctx, abi.FMT_INT8_IQ, fs, 0.0, [init], ring_samples=100 * 2048)
    trk.push(0, np.zeros(2 * 2048 * 80, np.int8))
    trk.run()
    ch = trk.channels()[0]
    assert ch.state == abi.IDLE
    assert trk.epoch_counts()[0] == abi.TrackingCfg.default().lock_fail_limit + 1


def test_code_advance_and_sample_accounting(ctx):
    """test_tracking.cpp:449-465."""
    fs = 2.048e6
    sv = ss.Sv(prn=7, cn0_dbhz=48.0, doppler_hz=-2200.0, delay_chips=100.25)
    raw = _raw(200, fs, [sv], "int8_iq", seed=79)
    init = _init(sv, fs, dop_err=100.0)
    trk = Tracker(ctx, abi.FMT_INT8_IQ, fs, 0.0, [init], ring_samples=300 * 2048, max_records=256)
    trk.push(0, raw.view(np.int8))
    trk.run()
    h = trk.records(0)
    assert len(h) >= 150
    for k in range(1, len(h)):
        assert abs((h[k]["chi_chips"] - h[k - 1]["chi_chips"]) - h[k - 1]["code_freq_hz"] / 1000.0) < 1e-9
    ch = trk.channels()[0]
    assert ch.sample_offset_next_epoch == h[0]["sample_offset_end"] + 2048 * (len(h) - 1)


def test_deterministic(ctx):
    """test_tracking.cpp:467-479: bitwise-identical reruns."""
    fs = 2.048e6
    sv = ss.Sv(prn=7, cn0_dbhz=45.0, doppler_hz=500.0, delay_chips=100.25)
    raw = _raw(300, fs, [sv], "int8_iq", seed=80)
    outs = []
    for _ in range(2):
        trk = Tracker(ctx, abi.FMT_INT8_IQ, fs, 0.0, [_init(sv, fs, dop_err=200.0)],
                      ring_samples=400 * 2048, max_records=300)
        trk.push(0, raw.view(np.int8))
        trk.run()
        outs.append(trk.records(0))
    assert outs[0].tobytes() == outs[1].tobytes()


def test_noop_kernel_closed_loop(ctx):
    """test_tracking.cpp:481-493."""
    fs = 2.048e6
    init = init_channel_from_acquisition(7, 1000.0, 0, 0, 0, fs)
    cf = init.code_freq_hz
    trk = Tracker(ctx, abi.FMT_INT8_IQ, fs, 0.0, [init], ring_samples=8 * 2048,
                  kernel=abi.KERNEL_NOOP)
    trk.push(0, np.tile(np.array([64, -32], np.int8), 2048))
    trk.run(max_epochs=1)
    r = trk.records(0)[0]
    assert r["ip"] == 0.0
    assert r["chi_chips"] == pytest.approx(cf / 1000.0, abs=1e-9)
    assert trk.channels()[0].sample_offset_next_epoch == 2048


def _batch_scenario(n_rec, fs, ms, seed):
    """Config 4 shape (scaled): independent recordings, 3 channels each."""
    rng = np.random.default_rng(seed)
    raws, inits, cstream, svs_all = [], [], [], []
    for r in range(n_rec):
        prns = rng.choice(np.arange(1, 33), 3, replace=False)
        svs = [ss.Sv(prn=int(p), cn0_dbhz=rng.uniform(38, 50), doppler_hz=rng.uniform(-5000, 5000),
                     delay_chips=rng.uniform(0, 1023)) for p in prns]
        raws.append(_raw(ms, fs, svs, "int16_iq", seed=seed * 100 + r))
        inits += [_init(sv, fs) for sv in svs]
        cstream += [r] * 3
        svs_all.append(svs)
    return np.stack(raws), inits, cstream


@pytest.mark.parametrize("mode", ["float2", "raw", "segment"])
def test_batched_recordings_throughput_mode(ctx, oracle_mod, mode):
    """Config 4 shape: recordings pushed in lock step (one strided H2D +
    one decode launch per chunk), narrow four-per-SM CTAs over float2 or raw
    cint16 rings, and the segment correlator (raw cint16 ring, per-warp TMA
    tensor copies, register captures); per-epoch replay parity for every
    channel, and the host and device strided pushes give bit-identical
    records."""
    import torch
    fs, ms, nrec = 65.472e6, 36, 4
    n = 65472
    raw, inits, cstream = _batch_scenario(nrec, fs, ms, seed=41)
    taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
    cfg = abi.TrackingCfg.default()
    chunk = 10 * n * 4

    def make():
        return Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, chan_stream=cstream, n_streams=nrec,
                       taps=taps, cfg=cfg, ring_samples=24 * n, max_records=ms,
                       cta_mode=abi.CTA_SEGMENT if mode == "segment" else abi.CTA_THROUGHPUT,
                       ring_raw=mode == "raw")
    a = make()
    for c0 in range(0, raw.shape[1], chunk):
        a.push_strided(raw[:, c0:c0 + chunk])
        a.run()
    b = make()
    dev = torch.from_numpy(raw).cuda()
    for c0 in range(0, raw.shape[1], chunk):
        k = min(chunk, raw.shape[1] - c0)
        b.push_device_strided(dev.data_ptr() + c0, k, raw.shape[1])
        b.run()
    b.sync()
    ca, cb = a.epoch_counts(), b.epoch_counts()
    assert np.array_equal(ca, cb) and ca.min() >= ms - 2
    att = None
    if mode == "segment":  # recordings attached in place: one launch, no ingest pass
        att = make()
        att.attach_device(dev.data_ptr(), raw.shape[1] // 4, raw.shape[1])
        att.run()
        att.sync()
        assert np.array_equal(att.epoch_counts(), ca)
    for c in range(len(inits)):
        ra, ta = a.records(c, tap_sums=True)
        rb = b.records(c)
        assert ra.tobytes() == rb.tobytes()
        if att is not None:
            assert ra.tobytes() == att.records(c).tobytes()
        x = oracle_mod.ingest(raw[cstream[c]], abi.FMT_INT16_IQ, fs)
        replay_check(oracle_mod, inits[c], ra, x, n, cfg, taps, fs, tap_sums=ta)


@pytest.mark.parametrize("layout", ["uneven", "interleaved"])
def test_segment_gang_tickets_uneven_and_interleaved(ctx, oracle_mod, layout):
    """The segment correlator's gang tickets (work drawn per recording by
    CTAs of one warp-slot class): recordings with 5, 1 and 3 channels (a
    ticket's spare members are skipped), and channels of three recordings
    interleaved (every gang a single channel: the plain item queue); 40
    epochs in work items of 16 (several chunks per channel); per-epoch replay
    parity and the attached run equal to the pushed one byte for byte."""
    import torch
    fs, ms, n = 65.472e6, 40, 65472
    rng = np.random.default_rng(97)
    per = [5, 1, 3] if layout == "uneven" else [3, 3, 3]
    raws, inits, cstream = [], [], []
    for r, k in enumerate(per):
        prns = rng.choice(np.arange(1, 33), k, replace=False)
        svs = [ss.Sv(prn=int(p), cn0_dbhz=rng.uniform(40, 50), doppler_hz=rng.uniform(-5000, 5000),
                     delay_chips=rng.uniform(0, 1023)) for p in prns]
        raws.append(_raw(ms, fs, svs, "int16_iq", seed=970 + r))
        inits += [_init(sv, fs) for sv in svs]
        cstream += [r] * k
    if layout == "interleaved":
        order = [0, 3, 6, 1, 4, 7, 2, 5, 8]
        inits = [inits[i] for i in order]
        cstream = [cstream[i] for i in order]
    raw = np.stack(raws)
    taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
    cfg = abi.TrackingCfg.default()

    def make():
        return Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, chan_stream=cstream, n_streams=len(per),
                       taps=taps, cfg=cfg, ring_samples=(ms + 4) * n, max_records=ms,
                       cta_mode=abi.CTA_SEGMENT)
    a = make()
    a.push_strided(raw)
    a.run()
    b = make()
    dev = torch.from_numpy(raw).cuda()
    b.attach_device(dev.data_ptr(), raw.shape[1] // 4, raw.shape[1])
    b.run()
    b.sync()
    ca = a.epoch_counts()
    assert np.array_equal(ca, b.epoch_counts()) and ca.min() >= ms - 2
    for c in range(len(inits)):
        ra, ta = a.records(c, tap_sums=True)
        assert ra.tobytes() == b.records(c).tobytes()
        x = oracle_mod.ingest(raw[cstream[c]], abi.FMT_INT16_IQ, fs)
        replay_check(oracle_mod, inits[c], ra, x, n, cfg, taps, fs, tap_sums=ta)


def test_bad_cta_mode_rejected(ctx):
    init = init_channel_from_acquisition(7, 0.0, 0, 0, 0, 2.048e6)
    with pytest.raises(ValueError):
        Tracker(ctx, abi.FMT_INT8_IQ, 2.048e6, 0.0, [init], ring_samples=8 * 2048, cta_mode=7)


def test_strided_push_rejects(ctx):
    fs, n = 2.048e6, 2048
    inits = [init_channel_from_acquisition(7, 0.0, 0, 0, 0, fs)] * 2
    trk = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, chan_stream=[0, 1], n_streams=2,
                  ring_samples=16 * n)
    with pytest.raises(ValueError):  # rows must match n_streams
        trk.push_strided(np.zeros((3, 4 * n), np.int16))
    trk.push(0, np.zeros(2 * n, np.int16))  # streams now out of step
    with pytest.raises(ValueError):
        trk.push_strided(np.zeros((2, 2 * n), np.int16))
    with pytest.raises(ValueError):  # larger than the ring
        trk2 = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, chan_stream=[0, 1], n_streams=2,
                       ring_samples=4 * n)
        trk2.push_strided(np.zeros((2, 2 * 8 * n), np.int16))


@pytest.mark.parametrize("K", [2, 3, 5, 12, 16])
def test_cluster_sizes(ctx, oracle_mod, K):
    """Each channel's epoch split over K CTAs (any K, not only powers of
    two): per-epoch replay parity, 4 channels of the config-2 shape."""
    fs, n = IF_FS, 16368
    rng = np.random.default_rng(20 + K)
    svs = [ss.Sv(prn=p, cn0_dbhz=rng.uniform(38, 50), doppler_hz=rng.uniform(-5000, 5000),
                 delay_chips=rng.uniform(0, 1023)) for p in (3, 8, 14, 27)]
    raw = _raw(80, fs, svs, "int8_real_if", IF_HZ, seed=30 + K)
    inits = [_init(sv, fs) for sv in svs]
    cfg, taps = abi.TrackingCfg.default(), abi.Taps.epl(0.5)
    trk = Tracker(ctx, abi.FMT_INT8_REAL_IF, fs, IF_HZ, inits, ring_samples=100 * n,
                  max_records=80, cta_mode=abi.CTA_LATENCY, cluster_size=K)
    trk.push(0, raw)
    trk.run()
    x = oracle_mod.ingest(raw, abi.FMT_INT8_REAL_IF, fs, IF_HZ)
    for c in range(len(inits)):
        recs = trk.records(c)
        assert len(recs) >= 77
        replay_check(oracle_mod, inits[c], recs, x, n, cfg, taps, fs)


@pytest.mark.parametrize("fmt,fs", [(abi.FMT_INT8_IQ, 2.048e6), (abi.FMT_INT16_IQ, 16.368e6)])
@pytest.mark.parametrize("cta_mode", [abi.CTA_AUTO, abi.CTA_SINGLE])
def test_raw_ring_matches_decoded_ring(ctx, oracle_mod, fmt, fs, cta_mode):
    """Raw complex-int rings (converted in the correlator with the decode
    scale folded into the rotators, a power of two) track like decoded
    float2 rings: both pass per-epoch replay parity, and with the same
    kernel (L1RXG_OVL=0: decoded latency-shape rings on track_kernel, as raw
    rings always are) the records are bit-identical.  (The overlapped kernel
    and the throughput shape's raw-ring tile size sum in another fp32 order.)"""
    n = int(round(fs / 1000))
    sv = ss.Sv(prn=7, cn0_dbhz=46.0, doppler_hz=-1500.0, delay_chips=321.7)
    name = "int8_iq" if fmt == abi.FMT_INT8_IQ else "int16_iq"
    raw = _raw(60, fs, [sv], name, seed=91)
    init = _init(sv, fs)
    cfg, taps = abi.TrackingCfg.default(), abi.Taps.epl(0.5)
    x = oracle_mod.ingest(raw, fmt, fs)
    outs = []
    for rr in (False, True):
        trk = Tracker(ctx, fmt, fs, 0.0, [init], ring_samples=70 * n, max_records=60,
                      cta_mode=cta_mode, ring_raw=rr)
        trk.push(0, raw)
        trk.run()
        outs.append(trk.records(0))
        assert len(outs[-1]) >= 58
        replay_check(oracle_mod, init, outs[-1], x, n, cfg, taps, fs)
    if os.environ.get("L1RXG_OVL") == "0":
        assert outs[0].tobytes() == outs[1].tobytes()


@pytest.mark.parametrize("env,sel", [
    ({"L1RXG_OVL": "0"}, "raw_ring_matches_decoded_ring or cluster_sizes"),
    ({"L1RXG_OVL_DWMAX": "-1"}, "cluster_sizes or odd_epoch_lengths or config1_shape or twelve_channel or multitap"),
    ({"L1RXG_OVL_RAWIF": "1"}, "config1_shape or twelve_channel or real_if_ring_wraps or cluster_sizes"),
], ids=["no_overlap", "overlap_exact_every_epoch", "raw_byte_ring_real_if"])
def test_latency_shape_variants(env, sel):
    """In a child process (the switches are read once per process): the
    non-overlapped kernel (L1RXG_OVL=0: raw-vs-decoded bit identity, replay
    parity), the overlapped kernel's exact phase-A recompute forced on
    every epoch (L1RXG_OVL_DWMAX=-1: replay parity through that path), and
    the real-IF stream as a raw byte ring filtered by the overlapped
    kernel's FIR warps (L1RXG_OVL_RAWIF=1; by default the ingest pass fills
    a float2 ring)."""
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_tracking.py"), "-k", sel],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("fs", [5.0e6, 3.969e6])
@pytest.mark.parametrize("cta_mode", [abi.CTA_AUTO, abi.CTA_SINGLE, abi.CTA_THROUGHPUT])
def test_odd_epoch_lengths(ctx, oracle_mod, fs, cta_mode):
    """Epoch lengths that are not multiples of the 31-sample run: 5 MHz (the
    paper's recordings, n = 5000) and n = 3969 (one sample past a full
    throughput tile: a 1-sample last unit, whose bulk copy has an empty first
    half), in every CTA shape; cint8 input, per-epoch replay parity."""
    n = int(round(fs / 1000))
    sv = ss.Sv(prn=21, cn0_dbhz=47.0, doppler_hz=2100.0, delay_chips=640.4)
    raw = _raw(50, fs, [sv], "int8_iq", seed=int(fs) % 1000)
    init = _init(sv, fs)
    cfg, taps = abi.TrackingCfg.default(), abi.Taps.epl(0.5)
    trk = Tracker(ctx, abi.FMT_INT8_IQ, fs, 0.0, [init], ring_samples=60 * n, max_records=50,
                  cta_mode=cta_mode)
    trk.push(0, raw.view(np.int8))
    trk.run()
    recs, tsums = trk.records(0, tap_sums=True)
    assert len(recs) >= 48
    x = oracle_mod.ingest(raw, abi.FMT_INT8_IQ, fs)
    replay_check(oracle_mod, init, recs, x, n, cfg, taps, fs, tap_sums=tsums)


@pytest.mark.parametrize("fs,tapset,ms", [(65.472e6, "wideband", 12), (65.472e6, "epl", 12),
                                          (16.368e6, "monitor", 8), (5.0e6, "epl", 12)])
def test_segment_correlator_ties_and_slow_paths(ctx, oracle_mod, fs, tapset, ms):
    """Segment correlator (cta_mode SEGMENT) per-epoch replay parity where
    its fast path does not apply.  First epoch at exactly commensurate NCO
    rates (Doppler 0, code rate 1.023 MHz: cps = 1/64 exactly at 65.472 MHz)
    and a half-chip code phase, so chip boundaries sit on exact fp64 ties;
    16 samples per chip with the 13-tap 0.1-chip monitor grid and 4.9
    samples per chip at 5 MHz (n = 5000, a partial last run) drive most runs
    through the exact per-sample slow path."""
    n = int(round(fs / 1000))
    if tapset == "wideband":
        taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
    elif tapset == "monitor":
        taps = abi.Taps.make([round(-0.5 + 0.1 * k, 10) for k in range(11)] + [0.25, -0.25],
                             early=11, prompt=5, late=12, n_counted=11)
    else:
        taps = abi.Taps.epl(0.5)
    svs = [ss.Sv(prn=9, cn0_dbhz=44.0, doppler_hz=0.0, delay_chips=12.5),
           ss.Sv(prn=17, cn0_dbhz=46.0, doppler_hz=-2750.0, delay_chips=411.3)]
    raw = _raw(ms + 2, fs, svs, "int16_iq", seed=23)
    inits = [_init(sv, fs) for sv in svs]
    assert inits[0].carrier_doppler_hz == 0.0 and inits[0].code_freq_hz == 1.023e6
    cfg = abi.TrackingCfg.default()
    trk = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, ring_samples=(ms + 4) * n, max_records=ms + 4,
                  taps=taps, cfg=cfg, cta_mode=abi.CTA_SEGMENT)
    trk.push(0, raw.view(np.int16))
    trk.run()
    x = oracle_mod.ingest(raw, abi.FMT_INT16_IQ, fs)
    for c, init in enumerate(inits):
        recs, tsums = trk.records(c, tap_sums=True)
        assert len(recs) >= ms - 2
        replay_check(oracle_mod, init, recs, x, n, cfg, taps, fs, tap_sums=tsums)


def test_segment_mode_rejects_other_formats(ctx):
    """The segment correlator takes complex int16 with enough samples per
    epoch for every warp of a CTA to own a unit (fs >= 3.073 MHz)."""
    init = init_channel_from_acquisition(7, 0.0, 0, 0, 0, 2.048e6)
    with pytest.raises(ValueError):
        Tracker(ctx, abi.FMT_INT8_IQ, 2.048e6, 0.0, [init], ring_samples=8 * 2048,
                cta_mode=abi.CTA_SEGMENT)
    init = init_channel_from_acquisition(7, 0.0, 0, 0, 0, 3.0e6)
    with pytest.raises(ValueError):
        Tracker(ctx, abi.FMT_INT16_IQ, 3.0e6, 0.0, [init], ring_samples=8 * 3000,
                cta_mode=abi.CTA_SEGMENT)


def test_segment_persistent_work_items(ctx, oracle_mod, monkeypatch):
    """The segment correlator's persistent CTAs take (chunk, channel) work
    items in order; a CTA that runs many items (grid capped to 3 CTAs) and
    chunks that wait for their predecessors give bit-identical records to the
    full grid; per-epoch replay parity on top."""
    import torch
    fs, ms, nrec = 65.472e6, 40, 3
    n = 65472
    raw, inits, cstream = _batch_scenario(nrec, fs, ms, seed=57)
    taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
    cfg = abi.TrackingCfg.default()
    dev = torch.from_numpy(raw).cuda()
    outs = []
    for grid in (None, "3"):
        if grid:
            monkeypatch.setenv("L1RXG_SEG_GRID", grid)
        trk = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, chan_stream=cstream, n_streams=nrec,
                      taps=taps, cfg=cfg, ring_samples=8 * n, max_records=ms, cta_mode=abi.CTA_SEGMENT)
        trk.attach_device(dev.data_ptr(), raw.shape[1] // 4, raw.shape[1])
        trk.run()
        trk.sync()
        outs.append([trk.records(c, tap_sums=True) for c in range(len(inits))])
        assert trk.epoch_counts().min() >= ms - 2
    monkeypatch.delenv("L1RXG_SEG_GRID", raising=False)
    for c in range(len(inits)):
        assert outs[0][c][0].tobytes() == outs[1][c][0].tobytes()
    x = oracle_mod.ingest(raw[cstream[0]], abi.FMT_INT16_IQ, fs)
    replay_check(oracle_mod, inits[0], outs[1][0][0], x, n, cfg, taps, fs, tap_sums=outs[1][0][1])


# ---- the CUDA scenario synthesizer (SimStream raw mode, l1rxg_simulate) ----

def _sim_svs():
    return [ss.Sv(prn=7, cn0_dbhz=48.0, doppler_hz=1200.0, delay_chips=61.38, phase0=0.3),
            ss.Sv(prn=12, cn0_dbhz=44.0, doppler_hz=-2600.0, delay_chips=500.25, phase0=1.1)]


@pytest.mark.parametrize("fmt", ["int16_iq", "int8_iq", "int8_real_if"])
def test_simulator_matches_torch_restatement_noise_free(ctx, fmt):
    """Noise-free bytes agree with the vectorised restatement (simsource.py)
    to one LSB (fp32 vs fp64 cos/sin at rounding ties only)."""
    fs, ms = 16.368e6, 6
    if_hz = 4.092e6 if fmt == "int8_real_if" else 0.0
    svs = _sim_svs()
    g = ss.synth_gpu(ctx, ms, fs, [svs], fmt=fmt, if_hz=if_hz, noise=False).cpu().numpy()[0]
    t = ss.synth(ms, fs, svs, fmt=fmt, if_hz=if_hz, noise=False, device="cuda").cpu().numpy()
    dt = np.int16 if fmt == "int16_iq" else np.int8
    a, b = g.view(dt).astype(np.int64), t.view(dt).astype(np.int64)
    d = np.abs(a - b)
    assert d.max() <= 1 and (d == 0).mean() > 0.999, (d.max(), (d == 0).mean())


def test_simulator_superposition_chunking_and_reproducibility(ctx):
    """test_simsource.cpp:80-119 properties: a two-SV stream is the sum of the
    single-SV streams (noise-free, within quantisation); fixed-seed bytes are
    reproducible and independent of chunking (ms0); recordings differ."""
    fs, ms = 16.368e6, 4
    svs = _sim_svs()
    both = ss.synth_gpu(ctx, ms, fs, [svs], noise=False).cpu().numpy()[0].view(np.int16).astype(np.int64)
    one = ss.synth_gpu(ctx, ms, fs, [svs[:1]], noise=False).cpu().numpy()[0].view(np.int16).astype(np.int64)
    two = ss.synth_gpu(ctx, ms, fs, [svs[1:]], noise=False).cpu().numpy()[0].view(np.int16).astype(np.int64)
    assert np.abs(both - (one + two)).max() <= 1
    a = ss.synth_gpu(ctx, ms, fs, [svs, svs], seed=77).cpu().numpy()
    b = ss.synth_gpu(ctx, ms, fs, [svs, svs], seed=77).cpu().numpy()
    assert a.tobytes() == b.tobytes()
    assert a[0].tobytes() != a[1].tobytes()  # noise keyed by recording
    c0 = ss.synth_gpu(ctx, 1, fs, [svs, svs], seed=77, ms0=0).cpu().numpy()
    c1 = ss.synth_gpu(ctx, ms - 1, fs, [svs, svs], seed=77, ms0=1).cpu().numpy()
    assert np.concatenate([c0, c1], axis=1).tobytes() == a.tobytes()


@pytest.mark.parametrize("fmt,fs", [("int16_iq", 16.368e6), ("int8_iq", 16.368e6), ("int16_iq", 65.472e6)])
def test_simulator_bytes_match_reference_simstream(ctx, oracle_mod, fmt, fs):
    """Byte-level parity with the reference simulator itself: the unmodified
    SimStream (simsource.hpp:253-331, oracle/_ref) renders the same noise-free
    satellites, quantised as generate_recording does (lround, clamp to
    +-127 / +-32767, simsource.hpp:393-413); the CUDA generator's bytes equal
    them except at rounding ties of its fp32 cos/sin (at most one LSB)."""
    if not oracle_mod.ref_available():
        pytest.skip("reference build absent")
    ms = 4
    svs = _sim_svs()
    g = ss.synth_gpu(ctx, ms, fs, [svs], fmt=fmt, noise=False).cpu().numpy()[0]
    ref = oracle_mod.ref_sim_baseband(
        [dict(prn=sv.prn, cn0=sv.cn0_dbhz, doppler=sv.doppler_hz, doppler_rate=sv.doppler_rate,
              delay_chips=sv.delay_chips, phase0=sv.phase0) for sv in svs], ms / 1000.0, fs, False, 0)
    scale, lim, dt = (32768.0, 32767, np.int16) if fmt == "int16_iq" else (128.0, 127, np.int8)
    v = np.stack([ref.real, ref.imag], -1).reshape(-1) * scale
    want = np.clip(np.sign(v) * np.floor(np.abs(v) + 0.5), -lim, lim).astype(np.int64)  # std::lround
    got = g.view(dt).astype(np.int64)
    assert got.size == want.size
    d = np.abs(got - want)
    assert d.max() <= 1 and (d == 0).mean() > 0.999, (d.max(), (d == 0).mean())


def test_simulator_noise_and_post_correlation_snr(ctx):
    """Noise of sigma/sqrt(2) per component (simsource.hpp:325-327) and the
    post-correlation SNR over 1 ms = C/N0 - 30 dB (test_simsource.cpp:149-179),
    measured with the GPU correlator (open-loop batch at the true code phase)."""
    fs, ms, cn0 = 5e6, 400, 45.0
    n = 5000
    noise_only = ss.synth_gpu(ctx, 50, fs, [[ss.Sv(prn=7, cn0_dbhz=-200.0)]], seed=3).cpu().numpy()[0]
    v = noise_only.view(np.int16).astype(np.float64) / 32768.0
    assert abs(v.std() - 0.25 / math.sqrt(2.0)) < 0.002 and abs(v.mean()) < 1e-3
    raw = ss.synth_gpu(ctx, ms, fs, [[ss.Sv(prn=7, cn0_dbhz=cn0)]], seed=2024).cpu().numpy()[0]
    iq = raw.view(np.int16).astype(np.float64) / 32768.0
    x = (iq[0::2] + 1j * iq[1::2]).reshape(ms, n)
    taps = abi.Taps.epl(0.5)
    st = [abi.Nco(0.0, 1.023e6, 0.0, 0.0, 0.0) for _ in range(ms)]
    sums, _ = ctx.correlate_batch(x, st, [7] * ms, taps, fs)
    p = sums[:, 2 * taps.prompt] + 1j * sums[:, 2 * taps.prompt + 1]
    m = p.mean()
    snr = 10 * math.log10(abs(m) ** 2 / (np.abs(p - m) ** 2).sum() * (len(p) - 1))
    assert abs(snr - (cn0 - 30.0)) < 1.0, snr


def test_auto_picks_segment_correlator_for_many_channels(ctx):
    """cta_mode AUTO with >= 2 x SMs channels of complex int16 at 64 samples
    per chip on the 0.25-chip grid selects the segment correlator: records
    bit-identical to an explicit CTA_SEGMENT tracker."""
    import torch
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    fs, ms = 65.472e6, 5
    nrec = (2 * nsm + 11) // 12
    rng = np.random.default_rng(5)
    raws, inits, cstream = [], [], []
    for r in range(nrec):
        prns = rng.choice(np.arange(1, 33), 12, replace=False)
        svs = [ss.Sv(prn=int(p), cn0_dbhz=45.0, doppler_hz=rng.uniform(-4000, 4000),
                     delay_chips=rng.uniform(0, 1023)) for p in prns]
        inits += [_init(sv, fs) for sv in svs]
        cstream += [r] * 12
        raws.append(svs)
    dev = ss.synth_gpu(ctx, ms, fs, raws, seed=9)
    taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
    outs = []
    for mode in (abi.CTA_AUTO, abi.CTA_SEGMENT):
        trk = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, chan_stream=cstream, n_streams=nrec, taps=taps,
                      ring_samples=(ms + 4) * 65472, max_records=ms, cta_mode=mode)
        trk.attach_device(dev.data_ptr(), dev.shape[1] // 4, dev.shape[1])
        trk.run()
        trk.sync()
        outs.append([trk.records(c) for c in range(len(inits))])  # the valid records only
    for a_, b_ in zip(*outs):
        assert len(a_) >= ms - 1 and a_.tobytes() == b_.tobytes()


def test_segment_max_epochs_and_noop(ctx, oracle_mod):
    """Segment correlator: run(max_epochs) in pieces gives the same records
    as one run (the persistent work items honour the epoch budget), and the
    Noop kernel advances the NCO only (test_tracking.cpp:481-493)."""
    fs, ms, n = 65.472e6, 12, 65472
    svs = [[ss.Sv(prn=5, cn0_dbhz=46.0, doppler_hz=900.0, delay_chips=40.5),
            ss.Sv(prn=23, cn0_dbhz=44.0, doppler_hz=-1700.0, delay_chips=800.0)]]
    dev = ss.synth_gpu(ctx, ms, fs, svs, seed=31)
    inits = [_init(sv, fs) for sv in svs[0]]
    taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)

    def make(kernel=abi.KERNEL_BATCHED):
        t = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, taps=taps, ring_samples=(ms + 4) * n,
                    max_records=ms, cta_mode=abi.CTA_SEGMENT, kernel=kernel)
        t.attach_device(dev.data_ptr(), dev.shape[1] // 4, dev.shape[1])
        return t
    one = make()
    one.run()
    pieces = make()
    for _ in range(6):
        pieces.run(max_epochs=3)
    assert np.array_equal(one.epoch_counts(), pieces.epoch_counts())
    for c in range(2):
        assert one.records(c).tobytes() == pieces.records(c).tobytes()
    noop = make(abi.KERNEL_NOOP)
    noop.run(max_epochs=4)
    r = noop.records(0)
    assert len(r) == 4 and np.all(r["ip"] == 0.0)
    for k in range(1, 4):
        assert abs((r[k]["chi_chips"] - r[k - 1]["chi_chips"]) - r[k - 1]["code_freq_hz"] / 1000.0) < 1e-9


def test_attach_refuses_pushes_and_detach_restores_ring(ctx):
    """Attached recordings are the rings: every push entry point is refused
    while they are attached (the kernel reads the attachment, so a push would
    silently advance availability past it), reset keeps the attachment with
    every sample available, and detach hands the tracker its own ring back."""
    import torch
    fs, ms, n = 65.472e6, 6, 65472
    svs = [[ss.Sv(prn=5, cn0_dbhz=46.0, doppler_hz=900.0, delay_chips=40.5)]]
    dev = ss.synth_gpu(ctx, ms, fs, svs, seed=33)
    inits = [_init(sv, fs) for sv in svs[0]]
    taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
    t = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, taps=taps, ring_samples=(ms + 4) * n,
                max_records=ms, cta_mode=abi.CTA_SEGMENT)
    t.attach_device(dev.data_ptr(), dev.shape[1] // 4, dev.shape[1])
    host = dev.cpu().numpy()
    with pytest.raises(ValueError, match="attached"):
        t.push(0, host[0, : 4 * n])
    with pytest.raises(ValueError, match="attached"):
        t.push_device(0, dev.data_ptr(), 4 * n)
    with pytest.raises(ValueError, match="attached"):
        t.push_strided(host[:, : 4 * n])
    with pytest.raises(ValueError, match="attached"):
        t.push_device_strided(dev.data_ptr(), 4 * n, dev.shape[1])
    t.run()
    first = t.records(0)
    t.reset(inits)  # the attachment stays: same records again
    t.run()
    assert t.records(0).tobytes() == first.tobytes()
    t.reset()  # the creation-time channels, restored on the device
    t.run()
    assert t.records(0).tobytes() == first.tobytes()
    t.detach()
    t.reset(inits)
    t.push(0, host[0])  # now into the ring: the same samples, the same records
    t.run()
    assert t.records(0).tobytes() == first.tobytes()


def test_segment_quarter_grid_start_chips_bit_identical(ctx, oracle_mod, monkeypatch):
    """On the quarter grid (every tap offset k/4 chip) three formulations give
    byte-identical records: the direct quarter-crossing kernel (default: every
    run locates its own crossings, no step table), the step-table kernel with
    the start-chip LUT (L1RXG_SEG_QDIRECT=0) and the step-table kernel with
    the exact per-tap fp64 start chips (L1RXG_SEG_QGRID=0) -- including at
    Doppler offsets that walk the code phase across quarter-chip boundaries."""
    fs, ms, n = 65.472e6, 30, 65472
    svs = [[ss.Sv(prn=p, cn0_dbhz=45.0, doppler_hz=dop, delay_chips=dl)
            for p, dop, dl in ((4, 4999.0, 100.25), (15, -3700.0, 512.5), (28, 120.0, 1000.75))]]
    dev = ss.synth_gpu(ctx, ms, fs, svs, seed=44)
    inits = [_init(sv, fs) for sv in svs[0]]
    taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
    out = []
    for qd, qg in (("1", "1"), ("0", "1"), ("0", "0")):
        monkeypatch.setenv("L1RXG_SEG_QDIRECT", qd)
        monkeypatch.setenv("L1RXG_SEG_QGRID", qg)
        t = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, taps=taps, ring_samples=(ms + 4) * n,
                    max_records=ms, cta_mode=abi.CTA_SEGMENT)
        t.attach_device(dev.data_ptr(), dev.shape[1] // 4, dev.shape[1])
        t.run()
        out.append([t.records(c, tap_sums=True) for c in range(3)])
    for other in out[1:]:
        for (ra, sa), (rb, sb) in zip(out[0], other):
            assert ra.tobytes() == rb.tobytes() and sa.tobytes() == sb.tobytes()
    x = oracle_mod.ingest(dev.cpu().numpy()[0], abi.FMT_INT16_IQ, fs)
    for c in range(3):
        replay_check(oracle_mod, inits[c], out[0][c][0], x, n, abi.TrackingCfg.default(), taps, fs,
                     tap_sums=out[0][c][1])


@pytest.mark.parametrize("cta_mode", [abi.CTA_AUTO, abi.CTA_SEGMENT])
def test_long_cn0_window_replay(ctx, oracle_mod, cta_mode):
    """cn0_window_ms beyond the POD's 64-entry window arrays (the reference
    allows any value >= 2, tracking.hpp:55-56): the device carries the window
    as running sums accumulated in push order; every epoch replays against the
    oracle (whose own window equals the reference's, test_oracle.py), C/N0 and
    the lock-fail counting included."""
    cfg = abi.TrackingCfg.default()
    cfg.cn0_window_ms = 100
    if cta_mode == abi.CTA_SEGMENT:
        fs, n, fmt, tag = 65.472e6, 65472, abi.FMT_INT16_IQ, "int16_iq"
        taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
        ms = 260
    else:
        fs, n, fmt, tag = IF_FS, 16368, abi.FMT_INT8_REAL_IF, "int8_real_if"
        taps = abi.Taps.epl(0.5)
        ms = 400
    sv = ss.Sv(prn=11, cn0_dbhz=44.0, doppler_hz=-1800.0, delay_chips=222.2)
    raw = _raw(ms, fs, [sv], tag, IF_HZ if tag == "int8_real_if" else 0.0, seed=91)
    init = _init(sv, fs)
    trk = Tracker(ctx, fmt, fs, IF_HZ if tag == "int8_real_if" else 0.0, [init], taps=taps, cfg=cfg,
                  ring_samples=(ms + 8) * n, max_records=ms, cta_mode=cta_mode)
    trk.push(0, raw)
    trk.run()
    recs, ts = trk.records(0, tap_sums=True)
    assert len(recs) >= ms - 2 and np.count_nonzero(recs["cn0_dbhz"]) > 0
    x = oracle_mod.ingest(raw, fmt, fs, IF_HZ if tag == "int8_real_if" else 0.0)
    replay_check(oracle_mod, init, recs, x, n, cfg, taps, fs, tap_sums=ts)
