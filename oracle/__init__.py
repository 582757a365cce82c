"""oracle -- TEST INFRASTRUCTURE: the CPU checker for the GPU hot path.

Two libraries, both loaded with ctypes:

* ``port``  -- oracle/lib/libl1rx_oracle.so, the plain-C restatement of the
  reference's tracking path (oracle/l1rx_oracle.c);
* ``ref``   -- oracle/_ref/libl1rx_ref.so, the UNMODIFIED reference headers
  (/root/reference/proj/include) compiled in place behind ref_shim.cpp;
* ``acq``   -- oracle/_ref/libl1rx_acq_ref.so, the unmodified reference
  acquisition (acquisition.hpp, fft.hpp) behind acq_shim.cpp with FFTW's
  API served by cuFFTW (executing a transform needs a GPU).
  Built only where /root/reference exists; the prebuilt .so travels to the
  GPU box with the gpurun snapshot.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package.  The product (paper_1907_00463_b200, libl1rxg.so) never
does: it fails loudly when its CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from functools import lru_cache

import numpy as np

from paper_1907_00463_b200.abi import (Channel, Corr, EpochRecord, Nco, Taps,
                                       TrackingCfg)

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "lib", "libl1rx_oracle.so")
REF_DIR = os.path.join(HERE, "_ref")
REF_INC = "/root/reference/proj/include"

_dp = C.POINTER(C.c_double)
_i8p = C.POINTER(C.c_int8)


def build(force: bool = False) -> None:
    """Builds the oracle C library, and _ref when the reference is present."""
    targets = ["lib/libl1rx_oracle.so"]
    if os.path.isdir(REF_INC):
        targets.append("ref")
    if force or not os.path.exists(PORT_SO) or (os.path.isdir(REF_INC) and not all(
            os.path.exists(os.path.join(REF_DIR, f)) for f in ("libl1rx_ref.so", "libl1rx_acq_ref.so"))):
        subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def ref_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libl1rx_ref.so"))


@lru_cache(maxsize=None)
def ref_path() -> str:
    """The -march=native reference build if this host has every ISA flag of
    the build host, else the x86-64-v3 build."""
    native = os.path.join(REF_DIR, "libl1rx_ref.so")
    v3 = os.path.join(REF_DIR, "libl1rx_ref_v3.so")
    fl = os.path.join(REF_DIR, "build_cpu_flags.txt")
    if os.path.exists(fl):
        with open(fl) as f:
            want = set(f.read().split(":", 1)[-1].split())
        isa = {x for x in want if x.startswith(("avx", "fma", "bmi", "sse", "amx", "f16c"))}
        if not isa <= _cpu_flags() and os.path.exists(v3):
            return v3
    return native


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


@lru_cache(maxsize=None)
def port():
    if not os.path.exists(PORT_SO):
        build()
    lib = C.CDLL(PORT_SO)
    P = C.POINTER
    _sig(lib, "orc_last_error", C.c_char_p)
    _sig(lib, "orc_ca_code", C.c_int, C.c_int, _i8p)
    _sig(lib, "orc_resample_code", C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, _i8p)
    _sig(lib, "orc_halfband_taps", None, _dp)
    _sig(lib, "orc_ingest_state_size", C.c_int)
    _sig(lib, "orc_ingest_init", None, C.c_void_p, C.c_int, C.c_double, C.c_double)
    _sig(lib, "orc_ingest", C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, _dp)
    _sig(lib, "orc_correlate", C.c_int, C.c_int, _dp, C.c_int, P(Nco), C.c_int, P(Taps),
         C.c_double, _dp, P(Corr))
    _sig(lib, "orc_track_epoch", C.c_int, P(Channel), _dp, C.c_int, P(TrackingCfg), P(Taps),
         C.c_double, C.c_int, P(EpochRecord), _dp)
    _sig(lib, "orc_init_channel", None, P(Channel), C.c_int, C.c_double, C.c_int64, C.c_int,
         C.c_int64, C.c_double)
    _sig(lib, "orc_default_cfg", None, P(TrackingCfg))
    _sig(lib, "orc_dll_discriminator", C.c_double, P(Corr))
    _sig(lib, "orc_pll_discriminator", C.c_double, C.c_double, C.c_double)
    _sig(lib, "orc_fll_discriminator", C.c_double, *([C.c_double] * 5))
    _sig(lib, "orc_fll_discriminator_di", C.c_double, *([C.c_double] * 5))
    _sig(lib, "orc_carrier_aid", C.c_double, C.c_double, C.c_double)
    _sig(lib, "orc_loop_filter_update", C.c_double, _dp, _dp, P(C.c_int32), C.c_double,
         C.c_double, C.c_double, C.c_double)
    _sig(lib, "orc_update_quality_metrics", None, P(Channel), P(Corr), P(TrackingCfg))
    _sig(lib, "orc_track_run", C.c_int, P(Channel), P(C.c_int32), C.c_int, P(_dp), P(C.c_int64),
         C.c_int, P(TrackingCfg), P(Taps), C.c_double, C.c_int, C.c_int64, C.c_int,
         P(EpochRecord), _dp, P(C.c_int64))
    _sig(lib, "orc_search_grid", C.c_int, _dp, C.c_int, C.c_int, C.c_int, C.c_double, _dp,
         C.c_int, C.c_int, C.c_int, _dp)
    return lib


@lru_cache(maxsize=None)
def ref():
    path = ref_path()
    if not os.path.exists(path):
        raise FileNotFoundError("reference oracle not built: " + path)
    lib = C.CDLL(path)
    P = C.POINTER
    _sig(lib, "ref_last_error", C.c_char_p)
    _sig(lib, "ref_ca_code", C.c_int, C.c_int, _i8p)
    _sig(lib, "ref_halfband_taps", None, _dp)
    _sig(lib, "ref_read_source", C.c_int64, C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_int,
         _dp, C.c_int64)
    _sig(lib, "ref_validate_source", C.c_int, C.c_int, C.c_double, C.c_double, C.c_int)
    _sig(lib, "ref_correlate", C.c_int, C.c_int, _dp, C.c_int, P(Nco), C.c_int, C.c_double,
         C.c_double, P(Corr))
    _sig(lib, "ref_track_epoch", C.c_int, P(Channel), _dp, C.c_int, P(TrackingCfg), C.c_double,
         C.c_int, P(EpochRecord))
    _sig(lib, "ref_track_buffer", C.c_int64, P(Channel), _dp, C.c_int64, C.c_int, P(TrackingCfg),
         C.c_double, C.c_int, C.c_int64, P(EpochRecord))
    _sig(lib, "ref_init_channel", None, P(Channel), C.c_int, C.c_double, C.c_int64, C.c_int,
         C.c_int64, C.c_double)
    _sig(lib, "ref_default_cfg", None, P(TrackingCfg))
    _sig(lib, "ref_dll_discriminator", C.c_double, P(Corr))
    _sig(lib, "ref_pll_discriminator", C.c_double, C.c_double, C.c_double)
    _sig(lib, "ref_fll_discriminator", C.c_double, *([C.c_double] * 5))
    _sig(lib, "ref_fll_discriminator_di", C.c_double, *([C.c_double] * 5))
    _sig(lib, "ref_carrier_aid", C.c_double, C.c_double, C.c_double)
    _sig(lib, "ref_loop_filter_update", C.c_double, _dp, _dp, P(C.c_int), C.c_double, C.c_double,
         C.c_double, C.c_double)
    _sig(lib, "ref_sim_baseband", C.c_int64, C.c_int, P(C.c_int), _dp, _dp, _dp, _dp, _dp,
         C.c_double, C.c_double, C.c_int, C.c_uint64, _dp, C.c_int64)
    _sig(lib, "ref_bench_pipeline", C.c_int, C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_int,
         P(Channel), P(TrackingCfg), C.c_int, C.c_int, C.c_int64, _dp, _dp, P(C.c_int64),
         P(Channel))
    return lib


def acq_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libl1rx_acq_ref.so"))


@lru_cache(maxsize=None)
def acq():
    from paper_1907_00463_b200.abi import AcqResult
    path = os.path.join(REF_DIR, "libl1rx_acq_ref.so")
    if not os.path.exists(path):
        raise FileNotFoundError("reference acquisition not built: " + path)
    lib = C.CDLL(path)
    P = C.POINTER
    _sig(lib, "acq_last_error", C.c_char_p)
    _sig(lib, "acq_doppler_bins", C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, _dp, C.c_int)
    for f in ("acq_acquire_pcs", "acq_acquire_fast"):
        _sig(lib, f, C.c_int, _dp, C.c_int64, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
             C.c_int, C.c_double, P(AcqResult))
    _sig(lib, "acq_pcs_plane", C.c_int, _dp, C.c_int, C.c_int, C.c_double, _dp, C.c_int, _dp)
    _sig(lib, "acq_pick_peak", C.c_int, _dp, C.c_int, C.c_int, _dp, C.c_int, C.c_double, C.c_double,
         P(AcqResult))
    return lib


def ref_doppler_bins(dmin: float, dmax: float, step: float = 0.0, integration_ms: int = 4) -> np.ndarray:
    """doppler_bins (acquisition.hpp:38-50)."""
    out = np.zeros(4096)
    n = acq().acq_doppler_bins(dmin, dmax, step, integration_ms, dptr(out), out.size)
    if n < 0:
        _raise(-n, acq().acq_last_error())
    return out[:n].copy()


def ref_acquire_pcs(iq: np.ndarray, prn: int, fs: float, dmin: float, dmax: float, step: float,
                    integration_ms: int, threshold: float = 2.0, fast: bool = False):
    """acquire_pcs / acquire_fast (acquisition.hpp:189-262): AcqResult."""
    from paper_1907_00463_b200.abi import AcqResult
    iq = np.ascontiguousarray(iq, np.complex128)
    out = AcqResult()
    fn = acq().acq_acquire_fast if fast else acq().acq_acquire_pcs
    rc = fn(dptr(iq.view(np.float64)), iq.size, prn, fs, dmin, dmax, step, integration_ms, threshold,
            C.byref(out))
    _raise(rc, acq().acq_last_error())
    return out


def ref_pcs_plane(iq: np.ndarray, n_seg: int, prn: int, fs: float, bins) -> np.ndarray:
    """The acquire_pcs plane cells[bin][sample delay] (acquisition.hpp:196-219)."""
    iq = np.ascontiguousarray(iq, np.complex128)
    b = np.ascontiguousarray(bins, np.float64)
    N = int(round(fs / 1000))
    cells = np.zeros((b.size, N))
    rc = acq().acq_pcs_plane(dptr(iq.view(np.float64)), n_seg, prn, fs, dptr(b), b.size, dptr(cells))
    _raise(rc, acq().acq_last_error())
    return cells


def ref_pick_peak(cells: np.ndarray, bins, prn: int, fs: float, threshold: float = 2.0):
    """detail::pick_peak (acquisition.hpp:114-149) over a caller plane."""
    from paper_1907_00463_b200.abi import AcqResult
    cells = np.ascontiguousarray(cells, np.float64)
    b = np.ascontiguousarray(bins, np.float64)
    out = AcqResult()
    rc = acq().acq_pick_peak(dptr(cells.reshape(-1)), cells.shape[0], cells.shape[1], dptr(b), prn, fs,
                             threshold, C.byref(out))
    _raise(rc, acq().acq_last_error())
    return out


# ---- numpy conveniences -------------------------------------------------

def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def ca_code(prn: int, which: str = "port") -> np.ndarray:
    out = np.zeros(1023, np.int8)
    lib = port() if which == "port" else ref()
    fn = lib.orc_ca_code if which == "port" else lib.ref_ca_code
    rc = fn(prn, out.ctypes.data_as(_i8p))
    if rc:
        raise IndexError("PRN must be in 1..32")
    return out


def ingest(raw: np.ndarray, fmt: int, fs: float, if_hz: float = 0.0) -> np.ndarray:
    """Oracle ingest (samples.hpp:177-253) of a whole byte stream ->
    complex128 samples."""
    lib = port()
    st = C.create_string_buffer(lib.orc_ingest_state_size())
    lib.orc_ingest_init(st, fmt, fs, if_hz)
    raw = np.ascontiguousarray(raw).view(np.uint8)
    nmax = raw.size
    out = np.zeros(2 * nmax, np.float64)
    n = lib.orc_ingest(st, raw.ctypes.data_as(C.c_void_p), raw.size, dptr(out))
    return out[: 2 * n].view(np.complex128)


def ref_ingest(raw: np.ndarray, fmt: int, fs: float, if_hz: float = 0.0,
               block_ms: int = 1, tmpdir: str = "/tmp") -> np.ndarray:
    """The reference SampleSource (samples.hpp:114-265) over the same bytes."""
    import tempfile
    raw = np.ascontiguousarray(raw).view(np.uint8)
    with tempfile.NamedTemporaryFile(dir=tmpdir, suffix=".bin", delete=False) as f:
        f.write(raw.tobytes())
        path = f.name
    try:
        nmax = raw.size
        out = np.zeros(2 * nmax, np.float64)
        n = ref().ref_read_source(path.encode(), fmt, fs, if_hz, block_ms, dptr(out), nmax)
        if n < 0:
            raise ValueError(ref().ref_last_error().decode())
        return out[: 2 * n].view(np.complex128)
    finally:
        os.unlink(path)


def correlate(iq: np.ndarray, nco: Nco, prn: int, taps: Taps, fs: float,
              kernel: int = 0):
    """Oracle K-tap correlator; returns (Corr, tap_sums[2K], advanced Nco)."""
    iq = np.ascontiguousarray(iq, np.complex128)
    st = Nco.from_buffer_copy(nco)
    sums = np.zeros(2 * taps.n_taps, np.float64)
    out = Corr()
    rc = port().orc_correlate(kernel, dptr(iq.view(np.float64)), iq.size, C.byref(st), prn,
                              C.byref(taps), fs, dptr(sums), C.byref(out))
    _raise(rc, port().orc_last_error())
    return out, sums, st


def ref_correlate(iq: np.ndarray, nco: Nco, prn: int, el_spacing: float, fs: float,
                  kernel: int = 0):
    iq = np.ascontiguousarray(iq, np.complex128)
    st = Nco.from_buffer_copy(nco)
    out = Corr()
    rc = ref().ref_correlate(kernel, dptr(iq.view(np.float64)), iq.size, C.byref(st), prn,
                             el_spacing, fs, C.byref(out))
    _raise(rc, ref().ref_last_error())
    return out, st


def _raise(rc: int, msg) -> None:
    if rc == 0:
        return
    text = msg.decode() if isinstance(msg, bytes) else str(msg)
    if rc == 1:
        raise ValueError(text)
    if rc == 2:
        raise RuntimeError(text)
    if rc == 3:
        raise IndexError(text)
    raise OSError(text)


def track_epoch(ch: Channel, iq: np.ndarray, cfg: TrackingCfg, taps: Taps, fs: float,
                kernel: int = 0):
    iq = np.ascontiguousarray(iq, np.complex128)
    rec = EpochRecord()
    sums = np.zeros(2 * taps.n_taps, np.float64)
    rc = port().orc_track_epoch(C.byref(ch), dptr(iq.view(np.float64)), iq.size, C.byref(cfg),
                                C.byref(taps), fs, kernel, C.byref(rec), dptr(sums))
    _raise(rc, port().orc_last_error())
    return rec, sums


def init_channel(prn, doppler, acq_start, code_delay, start_offset, fs, which="port") -> Channel:
    ch = Channel()
    if which == "port":
        port().orc_init_channel(C.byref(ch), prn, doppler, acq_start, code_delay, start_offset, fs)
    else:
        ref().ref_init_channel(C.byref(ch), prn, doppler, acq_start, code_delay, start_offset, fs)
    return ch


def track_run(chans, chan_stream, streams, n: int, cfg: TrackingCfg, taps: Taps, fs: float,
              max_epochs: int, threads: int = 1, kernel: int = 0, records: bool = True):
    """Oracle closed loop for many channels over complex128 streams.
    Returns (channels, epochs_done, records[c][e] as numpy structured, tap_sums)."""
    from paper_1907_00463_b200.abi import record_dtype
    nc = len(chans)
    carr = (Channel * nc)(*chans)
    cs = (C.c_int32 * nc)(*chan_stream)
    streams = [np.ascontiguousarray(s, np.complex128) for s in streams]
    sp = (_dp * len(streams))(*[dptr(s.view(np.float64)) for s in streams])
    sl = (C.c_int64 * len(streams))(*[s.size for s in streams])
    done = (C.c_int64 * nc)()
    recs = np.zeros(nc * max_epochs, record_dtype()) if records else None
    sums = np.zeros(nc * max_epochs * 2 * taps.n_taps) if records else None
    port().orc_track_run(carr, cs, nc, sp, sl, n, C.byref(cfg), C.byref(taps), fs, kernel,
                         max_epochs, threads,
                         recs.ctypes.data_as(C.POINTER(EpochRecord)) if records else None,
                         dptr(sums) if records else None, done)
    out = [carr[i] for i in range(nc)]
    if records:
        recs = recs.reshape(nc, max_epochs)
        sums = sums.reshape(nc, max_epochs, 2 * taps.n_taps)
    return out, list(done), recs, sums


def ref_track_buffer(ch: Channel, iq: np.ndarray, n: int, cfg: TrackingCfg, fs: float,
                     kernel: int = 0, max_epochs: int = 1 << 40):
    from paper_1907_00463_b200.abi import record_dtype
    iq = np.ascontiguousarray(iq, np.complex128)
    cap = min(max_epochs, iq.size // n + 1)
    recs = np.zeros(cap, record_dtype())
    c2 = ch.copy()
    done = ref().ref_track_buffer(C.byref(c2), dptr(iq.view(np.float64)), iq.size, n,
                                  C.byref(cfg), fs, kernel, cap,
                                  recs.ctypes.data_as(C.POINTER(EpochRecord)))
    if done < 0:
        _raise(-done, ref().ref_last_error())
    return c2, recs[:done]


def search_grid(iq: np.ndarray, N: int, n_seg: int, prn: int, fs: float, bins, delay_step: int,
                n_delays: int) -> np.ndarray:
    iq = np.ascontiguousarray(iq, np.complex128)
    b = np.ascontiguousarray(bins, np.float64)
    plane = np.zeros((b.size, n_delays), np.float64)
    rc = port().orc_search_grid(dptr(iq.view(np.float64)), N, n_seg, prn, fs, dptr(b), b.size,
                                delay_step, n_delays, dptr(plane))
    _raise(rc, port().orc_last_error())
    return plane


def ref_sim_baseband(svs, duration_s: float, fs: float, noise: bool, seed: int) -> np.ndarray:
    """SimStream (simsource.hpp:198-378) complex baseband for raw-mode SVs:
    svs = list of dicts(prn, cn0, doppler, doppler_rate, delay_chips, phase0)."""
    k = len(svs)
    prns = (C.c_int * k)(*[s["prn"] for s in svs])

    def arr(key, default=0.0):
        return np.array([s.get(key, default) for s in svs], np.float64)
    cn0, dop, rate = arr("cn0", 45.0), arr("doppler"), arr("doppler_rate")
    dly, ph0 = arr("delay_chips"), arr("phase0")
    nmax = int(round(duration_s * 1000)) * int(round(fs / 1000)) + 16
    out = np.zeros(2 * nmax, np.float64)
    n = ref().ref_sim_baseband(k, prns, dptr(cn0), dptr(dop), dptr(rate), dptr(dly), dptr(ph0),
                               duration_s, fs, int(noise), seed, dptr(out), nmax)
    if n < 0:
        _raise(-n, ref().ref_last_error())
    return out[: 2 * n].view(np.complex128)
