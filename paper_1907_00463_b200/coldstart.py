"""GPU cold start: search grid -> detections -> channel hand-off -> tracking.

SURVEY.md 8(f) item 2 (GPU acquisition hand-off).  Mirrors the reference's
acquisition result and hand-off (acquisition.hpp:52-59 AcquisitionResult,
:114-149 pick_peak, tracking.hpp:622-650 init_channel_from_acquisition):
the config-5 grid (l1rxg_search_grid) evaluates the correlator bank on the
GPU, pick_peak applies the reference's peak / runner-up rule on the
half-chip delay grid, and every detection becomes a tracking channel that
starts at its code boundary in the same device-resident recording.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import abi
from .tracking import init_channel_from_acquisition, pick_peak, search_grid

CHIP_RATE_HZ = 1.023e6


@dataclass
class AcquisitionResult:
    """acquisition.hpp:52-59."""
    prn: int
    detected: bool
    ratio: float
    doppler_hz: float
    code_delay_samples: int
    code_delay_chips: float


def acquire(ctx, raw, fmt: int, fs: float, if_hz: float, n_blocks: int, prns, bins,
            threshold_ratio: float = 2.0, device_ptr: int | None = None):
    """acquire_pcs + pick_peak (acquisition.hpp:114-222) for every PRN over
    the first n_blocks 1-ms blocks, on the GPU grid (delays on the half-chip
    grid: code_delay_samples is a multiple of fs / 2.046 MHz)."""
    spc = int(round(fs / CHIP_RATE_HZ / 2.0))
    plane = search_grid(ctx, raw, fmt, fs, if_hz, n_blocks, prns, bins, device_ptr=device_ptr)
    out = []
    for i, p in enumerate(np.asarray(prns, dtype=int)):
        r = pick_peak(plane[i], bins, fs, delay_step=spc, prn=int(p), threshold_ratio=threshold_ratio)
        out.append(AcquisitionResult(prn=int(p), detected=bool(r.detected), ratio=float(r.ratio),
                                     doppler_hz=float(r.doppler_hz), code_delay_samples=int(r.code_delay_samples),
                                     code_delay_chips=float(r.code_delay_chips)))
    return out, plane


def handoff(results, fs: float, acq_buffer_start: int = 0, start_offset_samples: int = 0):
    """init_channel_from_acquisition for every detection (tracking.hpp:622-650)."""
    return [init_channel_from_acquisition(r.prn, r.doppler_hz, acq_buffer_start,
                                          r.code_delay_samples, start_offset_samples, fs)
            for r in results if r.detected]


__all__ = ["AcquisitionResult", "acquire", "handoff", "abi"]
