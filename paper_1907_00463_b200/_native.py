"""Loader for libl1rxg.so (the CUDA library behind include/l1rxg.h).

Fails loudly: a missing library or symbol raises instead of falling back to
any CPU path (there is none in the product)."""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

from . import abi

PKG = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("L1RXG_SO") or os.path.join(PKG, "_lib", "libl1rxg.so")  # override: experiments

# every symbol include/l1rxg.h declares (tests/test_abi.py checks the header
# against this list and the .so against both)
EXPORTS = [
    "l1rxg_abi_version", "l1rxg_last_error", "l1rxg_default_tracking_cfg", "l1rxg_epl_taps",
    "l1rxg_ca_code", "l1rxg_halfband_taps", "l1rxg_create", "l1rxg_destroy", "l1rxg_host_alloc",
    "l1rxg_host_free", "l1rxg_correlate_epoch", "l1rxg_correlate_batch", "l1rxg_tracker_create",
    "l1rxg_tracker_destroy", "l1rxg_tracker_push", "l1rxg_tracker_push_device",
    "l1rxg_tracker_push_strided", "l1rxg_tracker_push_device_strided", "l1rxg_tracker_attach_device",
    "l1rxg_tracker_detach", "l1rxg_tracker_run",
    "l1rxg_tracker_sync", "l1rxg_tracker_channels", "l1rxg_tracker_epoch_counts",
    "l1rxg_tracker_records", "l1rxg_tracker_records_raw", "l1rxg_tracker_reset",
    "l1rxg_tracker_stream", "l1rxg_tracker_read_samples",
    "l1rxg_tracker_timing", "l1rxg_search_grid", "l1rxg_search_grid_ex", "l1rxg_search_grid_timing", "l1rxg_simulate",
    "l1rxg_pick_peak", "l1rxg_init_channel",
]


class L1rxgError(OSError):
    pass


def _sig(L, name, res, *args):
    f = getattr(L, name)
    f.restype = res
    f.argtypes = list(args)


@lru_cache(maxsize=None)
def lib():
    if not os.path.exists(SO):
        raise L1rxgError(
            f"libl1rxg.so not built ({SO}); run `python -m paper_1907_00463_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(SO)
    P, vp, i64, dp = C.POINTER, C.c_void_p, C.c_int64, C.POINTER(C.c_double)
    _sig(L, "l1rxg_abi_version", C.c_int)
    _sig(L, "l1rxg_last_error", C.c_char_p)
    _sig(L, "l1rxg_default_tracking_cfg", None, P(abi.TrackingCfg))
    _sig(L, "l1rxg_epl_taps", None, C.c_double, P(abi.Taps))
    _sig(L, "l1rxg_ca_code", C.c_int, C.c_int, P(C.c_int8))
    _sig(L, "l1rxg_halfband_taps", None, dp)
    _sig(L, "l1rxg_create", C.c_int, C.c_int, P(vp))
    _sig(L, "l1rxg_destroy", C.c_int, vp)
    _sig(L, "l1rxg_host_alloc", C.c_int, vp, i64, P(vp))
    _sig(L, "l1rxg_host_free", C.c_int, vp, vp)
    _sig(L, "l1rxg_correlate_epoch", C.c_int, vp, C.c_int, dp, C.c_int, P(abi.Nco), C.c_int,
         C.c_double, C.c_double, P(abi.Corr))
    _sig(L, "l1rxg_correlate_batch", C.c_int, vp, dp, C.c_int, C.c_int, P(abi.Nco), P(C.c_int32),
         P(abi.Taps), C.c_double, dp, P(abi.Corr))
    _sig(L, "l1rxg_tracker_create", C.c_int, vp, P(abi.TrackerDesc), P(abi.Channel), P(C.c_int32),
         P(vp))
    _sig(L, "l1rxg_tracker_destroy", C.c_int, vp)
    _sig(L, "l1rxg_tracker_push", C.c_int, vp, C.c_int, vp, i64)
    _sig(L, "l1rxg_tracker_push_device", C.c_int, vp, C.c_int, vp, i64)
    _sig(L, "l1rxg_tracker_push_strided", C.c_int, vp, vp, i64, i64)
    _sig(L, "l1rxg_tracker_push_device_strided", C.c_int, vp, vp, i64, i64)
    _sig(L, "l1rxg_tracker_attach_device", C.c_int, vp, vp, i64, i64)
    _sig(L, "l1rxg_tracker_detach", C.c_int, vp)
    _sig(L, "l1rxg_tracker_run", C.c_int, vp, C.c_int)
    _sig(L, "l1rxg_tracker_sync", C.c_int, vp)
    _sig(L, "l1rxg_tracker_channels", C.c_int, vp, P(abi.Channel))
    _sig(L, "l1rxg_tracker_epoch_counts", C.c_int, vp, P(i64))
    _sig(L, "l1rxg_tracker_records", C.c_int, vp, C.c_int, i64, i64, P(abi.EpochRecord), dp)
    _sig(L, "l1rxg_tracker_records_raw", C.c_int, vp, vp, C.c_int, P(i64))
    _sig(L, "l1rxg_tracker_reset", C.c_int, vp, P(abi.Channel))
    _sig(L, "l1rxg_tracker_stream", vp, vp)
    _sig(L, "l1rxg_tracker_read_samples", C.c_int, vp, C.c_int, i64, i64, dp)
    _sig(L, "l1rxg_tracker_timing", C.c_int, vp, dp, dp, P(i64))
    _sig(L, "l1rxg_search_grid", C.c_int, vp, C.c_int, vp, C.c_int, i64, C.c_double, C.c_double,
         C.c_int, P(C.c_int32), C.c_int, dp, C.c_int, C.c_int, C.c_int, dp)
    _sig(L, "l1rxg_search_grid_ex", C.c_int, vp, C.c_int, vp, C.c_int, i64, C.c_double, C.c_double,
         C.c_int, vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int)
    _sig(L, "l1rxg_search_grid_timing", C.c_int, vp, dp, dp)
    _sig(L, "l1rxg_pick_peak", C.c_int, dp, C.c_int, C.c_int, dp, C.c_int, C.c_int, C.c_double, C.c_double,
         P(abi.AcqResult))
    _sig(L, "l1rxg_init_channel", C.c_int, C.c_int, C.c_double, i64, i64, i64, C.c_double, P(abi.Channel))
    _sig(L, "l1rxg_simulate", C.c_int, vp, vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, i64,
         C.c_int, C.c_uint64, C.c_int, vp, i64)
    if L.l1rxg_abi_version() != abi.ABI_VERSION:
        raise L1rxgError("libl1rxg ABI version mismatch")
    return L


def check(rc: int) -> None:
    """Maps an l1rxg_status to the Python analogue of the reference's
    exception (include/l1rxg.h)."""
    if rc == abi.OK:
        return
    msg = lib().l1rxg_last_error().decode(errors="replace")
    if rc == abi.EINVAL:
        raise ValueError(msg)
    if rc == abi.ELOGIC:
        raise RuntimeError(msg)
    if rc == abi.ERANGE:
        raise IndexError(msg)
    if rc == abi.ENOMEM:
        raise MemoryError(msg)
    raise L1rxgError(msg)
