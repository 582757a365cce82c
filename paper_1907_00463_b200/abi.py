"""ctypes mirror of include/l1rxg.h (the C ABI of libl1rxg.so).

Field order and widths follow the header exactly; tests/test_abi.py checks
sizes and offsets against the compiled library.  Each struct cites the
reference type it mirrors.
"""
from __future__ import annotations

import ctypes as C

ABI_VERSION = 2
CODE_LENGTH = 1023
MAX_TAPS = 16
WIN_MAX = 64

# l1rxg_status -> reference exception type (see include/l1rxg.h)
OK, EINVAL, ELOGIC, ERANGE, ECUDA, ENOMEM = range(6)

KERNEL_SCALAR, KERNEL_BATCHED, KERNEL_NOOP = 0, 1, 2          # tracking.hpp:60
FMT_INT8_IQ, FMT_INT16_IQ, FMT_INT8_REAL_IF, FMT_CF64 = 0, 1, 2, 3  # samples.hpp:22-26
IDLE, ACQUIRED, TRACKING = 0, 1, 2                             # tracking.hpp:59
CTA_AUTO, CTA_LATENCY, CTA_THROUGHPUT, CTA_SINGLE, CTA_SEGMENT = 0, 1, 2, 3, 4

BYTES_PER_SAMPLE = {FMT_INT8_IQ: 2, FMT_INT16_IQ: 4, FMT_INT8_REAL_IF: 1}  # samples.hpp:33-40


class Nco(C.Structure):
    """NCO fields of ChannelState (tracking.hpp:181-185)."""
    _fields_ = [("code_phase_chips", C.c_double), ("code_freq_hz", C.c_double),
                ("carrier_doppler_hz", C.c_double), ("carrier_phase_rad", C.c_double),
                ("chi_chips", C.c_double)]


class Corr(C.Structure):
    """CorrelatorOutputs (tracking.hpp:19-23)."""
    _fields_ = [(n, C.c_double) for n in
                ("ie", "qe", "ip", "qp", "il", "ql", "ip_h1", "qp_h1", "ip_h2", "qp_h2")] + [
        ("n_samples", C.c_int32), ("pad_", C.c_int32)]

    def as_tuple(self):
        return (self.ie, self.qe, self.ip, self.qp, self.il, self.ql,
                self.ip_h1, self.qp_h1, self.ip_h2, self.qp_h2)


class TrackingCfg(C.Structure):
    """TrackingConfig (tracking.hpp:25-45)."""
    _fields_ = [("epoch_ms", C.c_int32), ("pad0_", C.c_int32),
                ("el_spacing_chips", C.c_double), ("dll_bandwidth_hz", C.c_double),
                ("dll_damping", C.c_double), ("pll_bandwidth_hz", C.c_double),
                ("pll_damping", C.c_double), ("fll_bandwidth_hz", C.c_double),
                ("fll_pull_in_ms", C.c_int32), ("fll_coarse_ms", C.c_int32),
                ("cn0_window_ms", C.c_int32), ("lock_fail_limit", C.c_int32),
                ("cn0_drop_dbhz", C.c_double), ("carrier_lock_drop", C.c_double)]

    @classmethod
    def default(cls) -> "TrackingCfg":
        c = cls()
        c.epoch_ms = 1
        c.el_spacing_chips = 0.5
        c.dll_bandwidth_hz = 2.0
        c.dll_damping = 0.707
        c.pll_bandwidth_hz = 25.0
        c.pll_damping = 0.707
        c.fll_bandwidth_hz = 15.0
        c.fll_pull_in_ms = 400
        c.fll_coarse_ms = 100
        c.cn0_window_ms = 20
        c.lock_fail_limit = 50
        c.cn0_drop_dbhz = 28.0
        c.carrier_lock_drop = 0.6
        return c


class Taps(C.Structure):
    """Replica tap set; E/P/L = (+s/2, 0, -s/2) is the reference's
    (tracking.hpp:237,252-254); more taps are the builder's K-tap form."""
    _fields_ = [("n_taps", C.c_int32), ("n_counted", C.c_int32), ("early", C.c_int32),
                ("prompt", C.c_int32), ("late", C.c_int32), ("pad_", C.c_int32),
                ("offsets_chips", C.c_double * MAX_TAPS)]

    @classmethod
    def epl(cls, el_spacing: float = 0.5) -> "Taps":
        t = cls()
        t.n_taps = 3
        t.n_counted = 3
        t.early, t.prompt, t.late = 0, 1, 2
        hs = el_spacing / 2.0
        t.offsets_chips[0] = hs
        t.offsets_chips[1] = 0.0
        t.offsets_chips[2] = -hs
        return t

    @classmethod
    def make(cls, offsets, early: int, prompt: int, late: int,
             n_counted: int | None = None) -> "Taps":
        offsets = list(offsets)
        if not 1 <= len(offsets) <= MAX_TAPS:
            raise ValueError("1..16 taps")
        t = cls()
        t.n_taps = len(offsets)
        t.n_counted = len(offsets) if n_counted is None else n_counted
        t.early, t.prompt, t.late = early, prompt, late
        for k, d in enumerate(offsets):
            t.offsets_chips[k] = float(d)
        return t

    def offsets(self):
        return [self.offsets_chips[k] for k in range(self.n_taps)]


class Channel(C.Structure):
    """ChannelState (tracking.hpp:177-207) as POD, minus NavDecodeState."""
    _fields_ = [("prn", C.c_int32), ("state", C.c_int32),
                ("code_phase_chips", C.c_double), ("code_freq_hz", C.c_double),
                ("carrier_doppler_hz", C.c_double), ("carrier_phase_rad", C.c_double),
                ("chi_chips", C.c_double),
                ("dll_integrator", C.c_double), ("dll_prev_error", C.c_double),
                ("pll_integrator", C.c_double), ("pll_prev_error", C.c_double),
                ("dll_primed", C.c_int32), ("pll_primed", C.c_int32),
                ("fll_enabled", C.c_int32), ("have_last_prompt", C.c_int32),
                ("last_ip", C.c_double), ("last_qp", C.c_double),
                ("epoch_ms_count", C.c_int64), ("epochs_since_handoff", C.c_int64),
                ("cn0_dbhz", C.c_double), ("carrier_lock_ratio", C.c_double),
                ("mu_smoothed", C.c_double),
                ("lock_fail_count", C.c_int32), ("metrics_valid", C.c_int32),
                ("sample_offset_next_epoch", C.c_int64),
                ("win_len", C.c_int32), ("pad_", C.c_int32),
                ("win_ip", C.c_double * WIN_MAX), ("win_qp", C.c_double * WIN_MAX)]

    def copy(self) -> "Channel":
        c = Channel()
        C.memmove(C.byref(c), C.byref(self), C.sizeof(Channel))
        return c

    def nco(self) -> Nco:
        return Nco(self.code_phase_chips, self.code_freq_hz, self.carrier_doppler_hz,
                   self.carrier_phase_rad, self.chi_chips)


class EpochRecord(C.Structure):
    """TrackingEpochOutput (tracking.hpp:209-222) + correlator in/out."""
    _fields_ = [("epoch_index", C.c_int64), ("sample_offset_start", C.c_int64),
                ("sample_offset_end", C.c_int64),
                ("prn", C.c_int32), ("state", C.c_int32), ("n_samples", C.c_int32),
                ("lock_fail_count", C.c_int32)] + [
        (n, C.c_double) for n in (
            "code_phase_in", "code_freq_in", "carrier_doppler_in", "carrier_phase_in",
            "ie", "qe", "ip", "qp", "il", "ql", "ip_h1", "qp_h1", "ip_h2", "qp_h2",
            "carrier_doppler_hz", "code_freq_hz", "code_phase_chips", "carrier_phase_rad",
            "chi_chips", "cn0_dbhz", "carrier_lock_ratio",
            "dll_integrator", "pll_integrator", "mu_smoothed",
            "dll_prev_error", "pll_prev_error")]


class TrackerDesc(C.Structure):
    _fields_ = [("format", C.c_int32), ("kernel", C.c_int32),
                ("sample_rate_hz", C.c_double), ("if_frequency_hz", C.c_double),
                ("n_streams", C.c_int32), ("n_channels", C.c_int32),
                ("ring_samples", C.c_int64), ("max_records", C.c_int32), ("cta_mode", C.c_int32),
                ("cluster_size", C.c_int32), ("ring_raw", C.c_int32),
                ("taps", Taps), ("cfg", TrackingCfg)]


class SimSv(C.Structure):
    """l1rxg_sim_sv: SimSatellite in raw mode (simsource.hpp:24-40)."""
    _fields_ = [("code_delay_chips", C.c_double), ("doppler_hz", C.c_double),
                ("doppler_rate_hz_per_s", C.c_double), ("initial_carrier_phase_rad", C.c_double),
                ("cn0_dbhz", C.c_double), ("prn", C.c_int32), ("pad_", C.c_int32)]


class AcqResult(C.Structure):
    """l1rxg_acq_result: AcquisitionResult (acquisition.hpp:52-59)."""
    _fields_ = [("prn", C.c_int32), ("detected", C.c_int32), ("ratio", C.c_double),
                ("doppler_hz", C.c_double), ("code_delay_samples", C.c_int32), ("pad_", C.c_int32),
                ("code_delay_chips", C.c_double)]


RECORD_DTYPE_FIELDS = [f[0] for f in EpochRecord._fields_]


def record_dtype():
    """numpy structured dtype identical to l1rxg_epoch_record."""
    import numpy as np
    m = {C.c_int64: "<i8", C.c_int32: "<i4", C.c_double: "<f8"}
    dt = np.dtype([(n, m[t]) for n, t in EpochRecord._fields_])
    assert dt.itemsize == C.sizeof(EpochRecord)
    return dt


def channel_array(chans):
    arr = (Channel * len(chans))()
    for i, c in enumerate(chans):
        arr[i] = c
    return arr
