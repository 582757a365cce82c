"""Host-side mirror of the reference tracking interface over libl1rxg.so.

Reference: /root/reference/proj/include/l1rx/tracking.hpp.  Names, argument
meaning and error behaviour follow the reference so the parity tests read
like its own tests:

=============================  ===========================================
reference (tracking.hpp)        here
=============================  ===========================================
CorrelatorOutputs  (:19-23)     abi.Corr
TrackingConfig     (:25-45)     abi.TrackingCfg  (TrackingConfig alias)
ChannelState       (:177-207)   abi.Channel      (ChannelState alias)
KernelKind         (:60)        KERNEL_SCALAR / KERNEL_BATCHED / KERNEL_NOOP
correlate_epoch_*  (:226-452)   correlate_epoch_gpu(view, ch, code, cfg, fs)
track_epoch        (:520-618)   Tracker (closed loop on device, per-epoch
                                records = TrackingEpochOutput)
ca_code_table      (cacode:99)  ca_code_table()
=============================  ===========================================

Error mapping (C++ exception -> Python): std::invalid_argument ->
ValueError, std::logic_error -> RuntimeError, std::out_of_range ->
IndexError, CUDA failures -> OSError.  There is no CPU fallback: if the
CUDA library or a GPU is missing, every compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import abi
from ._native import check, lib

ChannelState = abi.Channel
TrackingConfig = abi.TrackingCfg
CorrelatorOutputs = abi.Corr
KERNEL_SCALAR, KERNEL_BATCHED, KERNEL_NOOP = abi.KERNEL_SCALAR, abi.KERNEL_BATCHED, abi.KERNEL_NOOP

_dp = C.POINTER(C.c_double)


def llround(x: float) -> int:
    """std::llround: halves round away from zero (Python's round() rounds
    them to even; tracking.hpp:634 and pipeline.hpp:330 use llround)."""
    import math
    return int(math.copysign(math.floor(abs(x) + 0.5), x))


@dataclass
class CaCode:
    """CaCode (cacode.hpp:15-18)."""
    prn: int
    chips: np.ndarray  # int8, +/-1, length 1023


def generate_ca_code(prn: int) -> CaCode:
    """generate_ca_code (cacode.hpp:37-64), computed by libl1rxg."""
    out = np.zeros(1023, np.int8)
    check(lib().l1rxg_ca_code(prn, out.ctypes.data_as(C.POINTER(C.c_int8))))
    return CaCode(prn, out)


_TABLE = None


def ca_code_table():
    """ca_code_table (cacode.hpp:99-107): index 1..32."""
    global _TABLE
    if _TABLE is None:
        _TABLE = [CaCode(0, np.zeros(1023, np.int8))] + [generate_ca_code(p) for p in range(1, 33)]
    return _TABLE


class Context:
    """One device context (l1rxg_create)."""

    def __init__(self, device: int = 0):
        self._lib = lib()
        self.device = device
        p = C.c_void_p()
        check(self._lib.l1rxg_create(device, C.byref(p)))
        self.handle = p

    def close(self):
        if self.handle:
            self._lib.l1rxg_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def host_alloc(self, nbytes: int) -> np.ndarray:
        """Pinned host buffer (for the double-buffered H2D ingest ring)."""
        p = C.c_void_p()
        check(self._lib.l1rxg_host_alloc(self.handle, nbytes, C.byref(p)))
        buf = (C.c_uint8 * nbytes).from_address(p.value)
        arr = np.frombuffer(buf, np.uint8)
        arr_ptr = p.value
        ctx = self

        class _Pinned(np.ndarray):
            pass
        out = arr.view(_Pinned)
        import weakref
        weakref.finalize(out, lambda: ctx.handle and ctx._lib.l1rxg_host_free(ctx.handle, C.c_void_p(arr_ptr)))
        return out

    # ---- per-call compatibility path ---------------------------------
    def correlate_epoch(self, view, ch, prn: int, el_spacing: float, fs: float,
                        kernel: int = KERNEL_SCALAR) -> abi.Corr:
        """correlate_epoch_{scalar,batched,noop} contract: advances the NCO
        fields of ``ch`` (abi.Channel or abi.Nco) in place."""
        v = np.ascontiguousarray(view, np.complex128)
        nco = ch.nco() if isinstance(ch, abi.Channel) else ch
        out = abi.Corr()
        check(self._lib.l1rxg_correlate_epoch(self.handle, kernel,
                                              v.view(np.float64).ctypes.data_as(_dp), v.size,
                                              C.byref(nco), prn, el_spacing, fs, C.byref(out)))
        _store_nco(ch, nco)
        return out

    def correlate_batch(self, iq: np.ndarray, states, prns, taps: abi.Taps, fs: float):
        """Open-loop batch of independent channel-epochs.  iq: complex128
        [n_jobs, n]; states: list of abi.Nco (advanced in place).
        Returns (tap_sums [n_jobs, 2K], list of abi.Corr)."""
        iq = np.ascontiguousarray(iq, np.complex128)
        if iq.ndim == 1:
            iq = iq[None, :]
        nj, n = iq.shape
        st = (abi.Nco * nj)(*states)
        pr = (C.c_int32 * nj)(*[int(p) for p in prns])
        sums = np.zeros((nj, 2 * taps.n_taps), np.float64)
        corr = (abi.Corr * nj)()
        check(self._lib.l1rxg_correlate_batch(self.handle, iq.view(np.float64).ctypes.data_as(_dp),
                                              n, nj, st, pr, C.byref(taps), fs,
                                              sums.ctypes.data_as(_dp), corr))
        for k in range(nj):
            C.memmove(C.byref(states[k]), C.byref(st[k]), C.sizeof(abi.Nco))
        return sums, [corr[k] for k in range(nj)]


def search_grid(ctx: "Context", raw, fmt: int, fs: float, if_hz: float, n_blocks: int, prns, bins,
                n_delays: int | None = None, device_ptr: int | None = None, out=None,
                out_device_ptr: int | None = None, dtype=np.float64):
    """acquire_pcs plane semantics (acquisition.hpp:170-222) on the GPU:
    returns plane[prn][bin][delay] for delays d = k * (samples per half chip),
    cells N * |sum_n wiped[n] code[(n - d) mod N]| summed over n_blocks
    1-ms segments.  raw: host bytes, or device_ptr for bytes in HBM.  The
    plane lands in `out` (a host array, pinned is fastest) or at
    out_device_ptr (device memory), as float64 or float32 (`dtype`)."""
    spc = int(round(fs / 1.023e6 / 2.0))
    nd = n_delays or 2046
    prns = np.ascontiguousarray(prns, np.int32)
    bins = np.ascontiguousarray(bins, np.float64)
    f32 = np.dtype(dtype) == np.float32
    if device_ptr is not None:
        ptr, on_dev, nbytes = C.c_void_p(device_ptr), 1, int(raw)
    else:
        a = np.ascontiguousarray(raw).view(np.uint8)
        ptr, on_dev, nbytes = a.ctypes.data_as(C.c_void_p), 0, a.nbytes
    if out_device_ptr is not None:
        dst, dst_dev, plane = C.c_void_p(out_device_ptr), 1, None
    else:
        plane = out if out is not None else np.zeros((prns.size, bins.size, nd), np.float32 if f32 else np.float64)
        if plane.dtype != (np.float32 if f32 else np.float64) or plane.size != prns.size * bins.size * nd:
            raise ValueError("out: wrong dtype or size")
        dst, dst_dev = C.c_void_p(plane.ctypes.data), 0
    check(ctx._lib.l1rxg_search_grid_ex(ctx.handle, fmt, ptr, on_dev, nbytes, fs, if_hz, n_blocks,
                                        prns.ctypes.data_as(C.c_void_p), prns.size,
                                        bins.ctypes.data_as(C.c_void_p), bins.size, spc, nd, dst, int(f32),
                                        dst_dev))
    return plane.reshape(prns.size, bins.size, nd) if plane is not None else None


def search_grid_timing(ctx: "Context"):
    a, b = C.c_double(), C.c_double()
    check(ctx._lib.l1rxg_search_grid_timing(ctx.handle, C.byref(a), C.byref(b)))
    return a.value, b.value


def pick_peak(plane_row: np.ndarray, bins, fs: float, delay_step: int | None = None,
              prn: int = 0, threshold_ratio: float = 2.0) -> abi.AcqResult:
    """detail::pick_peak (acquisition.hpp:114-149) over one PRN's plane
    [bin][k] with delays d = k * delay_step samples (default: the search
    grid's half-chip step), by the library's l1rxg_pick_peak: the peak cell
    and the runner-up over every bin outside +-ceil(fs / chip rate) samples
    of the peak delay.  Returns AcquisitionResult (acquisition.hpp:52-59)."""
    cells = np.ascontiguousarray(plane_row, np.float64)
    b = np.ascontiguousarray(bins, np.float64)
    nb, nd = cells.shape
    step = delay_step if delay_step is not None else int(round(fs / 1.023e6 / 2.0))
    out = abi.AcqResult()
    check(lib().l1rxg_pick_peak(cells.ctypes.data_as(_dp), nb, nd, b.ctypes.data_as(_dp), step, prn, fs,
                                threshold_ratio, C.byref(out)))
    return out


def _store_nco(ch, nco: abi.Nco) -> None:
    ch.code_phase_chips = nco.code_phase_chips
    ch.code_freq_hz = nco.code_freq_hz
    ch.carrier_doppler_hz = nco.carrier_doppler_hz
    ch.carrier_phase_rad = nco.carrier_phase_rad
    ch.chi_chips = nco.chi_chips


_DEFAULT_CTX = {}


def default_context(device: int = 0) -> Context:
    if device not in _DEFAULT_CTX:
        _DEFAULT_CTX[device] = Context(device)
    return _DEFAULT_CTX[device]


def correlate_epoch_gpu(view, ch: abi.Channel, code: CaCode, cfg: abi.TrackingCfg,
                        sample_rate_hz: float) -> abi.Corr:
    """Drop-in for correlate_epoch_scalar/_batched (tracking.hpp:226-230,
    288-292): same arguments, same in-place state advance, same errors."""
    return default_context().correlate_epoch(view, ch, code.prn, cfg.el_spacing_chips,
                                             sample_rate_hz, KERNEL_SCALAR)


def correlate_epoch_noop(view, ch: abi.Channel, sample_rate_hz: float) -> abi.Corr:
    return default_context().correlate_epoch(view, ch, ch.prn or 1, 0.5, sample_rate_hz,
                                             KERNEL_NOOP)


class Tracker:
    """Closed-loop tracking of many channels over device sample rings.

    Replaces Receiver::tracking_round's per-channel track_epoch fan-out
    (pipeline.hpp:563-610) and SampleSource + BlockQueue ingest
    (samples.hpp:136-253, pipeline.hpp:388-404)."""

    def __init__(self, ctx: Context, fmt: int, fs: float, if_hz: float, channels,
                 chan_stream=None, n_streams: int = 1, taps: abi.Taps | None = None,
                 cfg: abi.TrackingCfg | None = None, kernel: int = KERNEL_SCALAR,
                 ring_samples: int | None = None, max_records: int = 1024,
                 cta_mode: int = abi.CTA_AUTO, cluster_size: int = 0, ring_raw: bool = False):
        self.ctx = ctx
        self._lib = ctx._lib
        self.fmt, self.fs, self.if_hz = fmt, fs, if_hz
        self.n = llround(fs / 1000.0)
        self.taps = taps or abi.Taps.epl(0.5)
        self.cfg = cfg or abi.TrackingCfg.default()
        chans = list(channels)
        self.n_channels = len(chans)
        d = abi.TrackerDesc()
        d.format, d.kernel = fmt, kernel
        d.sample_rate_hz, d.if_frequency_hz = fs, if_hz
        d.n_streams, d.n_channels = n_streams, len(chans)
        d.ring_samples = ring_samples or 64 * self.n
        d.max_records = max_records
        d.cta_mode = cta_mode
        d.cluster_size = cluster_size
        d.ring_raw = int(ring_raw)
        d.taps, d.cfg = self.taps, self.cfg
        self.desc = d
        cs = chan_stream if chan_stream is not None else [0] * len(chans)
        carr = (abi.Channel * max(1, len(chans)))(*chans)
        csarr = (C.c_int32 * max(1, len(chans)))(*cs)
        h = C.c_void_p()
        check(self._lib.l1rxg_tracker_create(ctx.handle, C.byref(d), carr, csarr, C.byref(h)))
        self.handle = h
        self.bps = abi.BYTES_PER_SAMPLE[fmt]

    def close(self):
        if self.handle:
            self._lib.l1rxg_tracker_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def push(self, stream: int, data) -> None:
        """Host bytes (numpy uint8/int8/int16 array; pinned is fastest)."""
        a = np.ascontiguousarray(data)
        check(self._lib.l1rxg_tracker_push(self.handle, stream, a.ctypes.data_as(C.c_void_p), a.nbytes))
        self._keep = a  # keep the source alive until the async copy is done

    def push_device(self, stream: int, dev_ptr: int, nbytes: int) -> None:
        check(self._lib.l1rxg_tracker_push_device(self.handle, stream, C.c_void_p(dev_ptr), nbytes))

    def push_strided(self, data: np.ndarray) -> None:
        """Host array [n_streams, k] (rows may be a column slice of a wider
        array): chunk k of every stream, one pitched copy + one launch."""
        if data.ndim != 2 or data.shape[0] != self.desc.n_streams or data.strides[1] != data.itemsize:
            raise ValueError("expected a [n_streams, k] array with contiguous rows")
        check(self._lib.l1rxg_tracker_push_strided(self.handle, C.c_void_p(data.ctypes.data),
                                                   data.shape[1] * data.itemsize, data.strides[0]))
        self._keep = data

    def attach_device(self, dev_ptr: int, samples_per_stream: int, stride_bytes: int) -> None:
        """Segment correlator only: complex-int16 recordings resident in device
        memory (stream s at dev_ptr + s * stride_bytes) become the rings; no
        ingest pass (l1rxg_tracker_attach_device)."""
        check(self._lib.l1rxg_tracker_attach_device(self.handle, C.c_void_p(dev_ptr),
                                                    C.c_int64(samples_per_stream), C.c_int64(stride_bytes)))

    def detach(self) -> None:
        """Ends an attachment: the tracker reads its own ring again and its
        streams restart empty (l1rxg_tracker_detach)."""
        check(self._lib.l1rxg_tracker_detach(self.handle))

    def push_device_strided(self, dev_ptr: int, nbytes_per_stream: int, stride_bytes: int) -> None:
        """Same-length chunk for every stream in one launch (batched recordings)."""
        check(self._lib.l1rxg_tracker_push_device_strided(self.handle, C.c_void_p(dev_ptr),
                                                          nbytes_per_stream, stride_bytes))

    def run(self, max_epochs: int = -1) -> None:
        check(self._lib.l1rxg_tracker_run(self.handle, max_epochs))

    def sync(self) -> None:
        check(self._lib.l1rxg_tracker_sync(self.handle))

    def channels(self):
        arr = (abi.Channel * max(1, self.n_channels))()
        check(self._lib.l1rxg_tracker_channels(self.handle, arr))
        return [arr[k] for k in range(self.n_channels)]

    def epoch_counts(self) -> np.ndarray:
        out = np.zeros(max(1, self.n_channels), np.int64)
        check(self._lib.l1rxg_tracker_epoch_counts(self.handle, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out[: self.n_channels]

    def records(self, channel: int, e0: int = 0, count: int | None = None, tap_sums: bool = False):
        """TrackingEpochOutput-like records (numpy structured array)."""
        if count is None:
            count = int(self.epoch_counts()[channel]) - e0
        recs = np.zeros(count, abi.record_dtype())
        sums = np.zeros((count, 2 * self.taps.n_taps), np.float64) if tap_sums else None
        check(self._lib.l1rxg_tracker_records(
            self.handle, channel, e0, count, recs.ctypes.data_as(C.POINTER(abi.EpochRecord)),
            sums.ctypes.data_as(_dp) if tap_sums else None))
        return (recs, sums) if tap_sums else recs

    def records_nbytes(self) -> int:
        """Bytes `records_raw` writes (every channel x max_records)."""
        nb = C.c_int64()
        check(self._lib.l1rxg_tracker_records_raw(self.handle, None, 0, C.byref(nb)))
        return nb.value

    def records_raw(self, dst_ptr: int | None = None, device: bool = False):
        nb = C.c_int64()
        check(self._lib.l1rxg_tracker_records_raw(self.handle, None, 0, C.byref(nb)))
        if dst_ptr is None:
            out = np.zeros(nb.value // C.sizeof(abi.EpochRecord), abi.record_dtype())
            check(self._lib.l1rxg_tracker_records_raw(self.handle, out.ctypes.data_as(C.c_void_p), 0,
                                                      C.byref(nb)))
            return out
        check(self._lib.l1rxg_tracker_records_raw(self.handle, C.c_void_p(dst_ptr), int(device),
                                                  C.byref(nb)))
        return nb.value

    def reset(self, channels=None) -> None:
        """Restart all streams at sample 0 with fresh channel states
        (channels=None: the ones given at creation, restored on the device)."""
        if channels is None:
            check(self._lib.l1rxg_tracker_reset(self.handle, None))
            return
        chans = list(channels)
        arr = (abi.Channel * max(1, len(chans)))(*chans)
        check(self._lib.l1rxg_tracker_reset(self.handle, arr))

    def cuda_stream(self) -> int:
        """cudaStream_t of the tracker's kernels (wrap with
        torch.cuda.ExternalStream to time with events)."""
        return int(self._lib.l1rxg_tracker_stream(self.handle) or 0)

    def read_samples(self, stream: int, s0: int, count: int) -> np.ndarray:
        out = np.zeros(2 * count, np.float64)
        check(self._lib.l1rxg_tracker_read_samples(self.handle, stream, s0, count, out.ctypes.data_as(_dp)))
        return out.view(np.complex128)

    def timing(self):
        """(ingest_ms, track_ms, kernel_launches) since the last call."""
        a, b, n = C.c_double(), C.c_double(), C.c_int64()
        check(self._lib.l1rxg_tracker_timing(self.handle, C.byref(a), C.byref(b), C.byref(n)))
        return a.value, b.value, n.value


def init_channel_from_acquisition(prn: int, doppler_hz: float, acq_buffer_start: int,
                                  code_delay_samples: int, start_offset_samples: int,
                                  sample_rate_hz: float) -> abi.Channel:
    """init_channel_from_acquisition (tracking.hpp:622-650) by the library's
    l1rxg_init_channel: host-side channel hand-off (once per channel)."""
    ch = abi.Channel()
    check(lib().l1rxg_init_channel(prn, doppler_hz, acq_buffer_start, code_delay_samples,
                                   start_offset_samples, sample_rate_hz, C.byref(ch)))
    return ch
