"""Seeded synthetic IF/baseband recordings for the benchmark configs.

Restates the signal model of the reference simulator's raw mode
(SimStream, simsource.hpp:194-378) in vectorised torch (CPU or CUDA):

* effective delay tau(t) = delay_chips / chip_rate - (fD t + rate t^2 / 2) / f_L1
  (simsource.hpp:344-352);
* per 1-ms block, chip count and carrier phase are interpolated linearly
  between the block edges (:269-284);
* amplitude A = sigma * sqrt(10^(CN0/10) / fs) with sigma = 0.25 complex
  noise (:237-239, :246, :324-327);
* quantisation lround/clamp to int8 / int16 (:393-413).

Builder extensions, NOT reference behaviour (the reference simulator emits
complex baseband only, simsource.hpp:421-423, and forbids duplicate PRNs,
:59-61):

* real-IF output Re{s(n) exp(+j 2 pi IF n / fs)} + N(0, sigma^2/4): after the
  receiver's mixer, half-band filter and x2 gain (samples.hpp:215-253) the
  in-band baseband noise density is sigma^2/fs again (total power sigma^2/2
  in the half band), so C/N0 is preserved up to the filter's ~1 dB
  signal-sidelobe loss (measured with the reference loops: 43.9 dB-Hz
  estimated at 45 dB-Hz, vs 44.9 for complex baseband);
* spoofed copies of a PRN summed as extra components (superposition,
  test_simsource.cpp:80-104).

Nav data is unmodulated (the reference's default without bits or
ephemeris, simsource.hpp:233-235).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .tracking import llround

CHIP_RATE = 1.023e6
F_L1 = 1.57542e9
NOISE_SIGMA = 0.25


@dataclass
class Sv:
    prn: int
    cn0_dbhz: float = 45.0
    doppler_hz: float = 0.0
    delay_chips: float = 0.0
    doppler_rate: float = 0.0
    phase0: float = 0.0


def _codes_table():
    # generate_ca_code (cacode.hpp:37-64) on the host, numpy
    taps = [(0, 0), (2, 6), (3, 7), (4, 8), (5, 9), (1, 9), (2, 10), (1, 8), (2, 9), (3, 10), (2, 3),
            (3, 4), (5, 6), (6, 7), (7, 8), (8, 9), (9, 10), (1, 4), (2, 5), (3, 6), (4, 7), (5, 8),
            (6, 9), (1, 3), (4, 6), (5, 7), (6, 8), (7, 9), (8, 10), (1, 6), (2, 7), (3, 8), (4, 9)]
    out = np.zeros((33, 1023), np.int8)
    for prn in range(1, 33):
        g1 = g2 = 0x3FF
        t1, t2 = taps[prn][0] - 1, taps[prn][1] - 1
        for i in range(1023):
            o = ((g1 >> 9) ^ (g2 >> t1) ^ (g2 >> t2)) & 1
            out[prn, i] = 1 - 2 * o
            f1 = ((g1 >> 2) ^ (g1 >> 9)) & 1
            f2 = ((g2 >> 1) ^ (g2 >> 2) ^ (g2 >> 5) ^ (g2 >> 7) ^ (g2 >> 8) ^ (g2 >> 9)) & 1
            g1 = ((g1 << 1) | f1) & 0x3FF
            g2 = ((g2 << 1) | f2) & 0x3FF
    return out


_CODES = None


def codes():
    global _CODES
    if _CODES is None:
        _CODES = _codes_table()
    return _CODES


def true_delay_s(sv: Sv, t):
    """Effective signal delay (simsource.hpp:346-352, raw mode)."""
    cycles = sv.doppler_hz * t + 0.5 * sv.doppler_rate * t * t
    return sv.delay_chips / CHIP_RATE - cycles / F_L1


def synth(n_ms: int, fs: float, svs, *, fmt: str = "int16_iq", if_hz: float = 0.0,
          seed: int = 1, device: str = "cpu", noise: bool = True, chunk_ms: int = 100,
          ms0: int = 0):
    """Returns the recording as a torch uint8 tensor of raw bytes
    (int8_iq / int16_iq little-endian / int8_real_if), on `device`.
    `ms0` starts the recording at that millisecond of the scenario (chunked
    generation of long recordings gives identical bytes per ms only when
    the same chunk boundaries are used; the noise stream is seeded per
    chunk from (seed, chunk index))."""
    import torch
    n = llround(fs / 1000.0)
    if abs(fs / 1000.0 - n) > 1e-9:
        raise ValueError("simulator requires an integer number of samples per ms")
    dev = torch.device(device)
    code_t = torch.as_tensor(codes().astype(np.float64), device=dev)
    chunks = []
    i = torch.arange(n, device=dev, dtype=torch.float64)
    for c0 in range(ms0, ms0 + n_ms, chunk_ms):
        nb = min(chunk_ms, ms0 + n_ms - c0)
        k = torch.arange(c0, c0 + nb, device=dev, dtype=torch.float64)[:, None]
        re = torch.zeros(nb, n, device=dev, dtype=torch.float64)
        im = torch.zeros_like(re)
        for sv in svs:
            amp = NOISE_SIGMA * math.sqrt(10.0 ** (sv.cn0_dbhz / 10.0) / fs) if noise else \
                math.sqrt(10.0 ** (sv.cn0_dbhz / 10.0) / fs)
            t0 = k * 1e-3
            t1 = t0 + 1e-3
            tau0 = true_delay_s(sv, t0)
            tau1 = true_delay_s(sv, t1)
            ch0 = (t0 + 6.0 - tau0) * CHIP_RATE  # off = tow_start - nav_encode_start = 6 s
            ch1 = (t1 + 6.0 - tau1) * CHIP_RATE
            chips = ch0 + i * ((ch1 - ch0) / n)
            ic = torch.floor(chips).to(torch.int64)
            chip = code_t[sv.prn][torch.remainder(ic, 1023)]
            th0 = sv.phase0 - 2.0 * math.pi * F_L1 * tau0
            th1 = sv.phase0 - 2.0 * math.pi * F_L1 * tau1
            th = th0 + i * ((th1 - th0) / n)
            re += amp * chip * torch.cos(th)
            im += amp * chip * torch.sin(th)
        g = torch.Generator(device=dev)
        g.manual_seed(int(seed) * 1000003 + c0)
        if fmt == "int8_real_if":
            gi = (torch.arange(c0 * n, (c0 + nb) * n, device=dev, dtype=torch.int64)).reshape(nb, n)
            ph = 2.0 * math.pi * if_hz / fs * gi.to(torch.float64)
            v = re * torch.cos(ph) - im * torch.sin(ph)
            if noise:
                v += (NOISE_SIGMA / 2.0) * torch.randn(nb, n, generator=g, device=dev,
                                                                  dtype=torch.float64)
            q = torch.clamp(torch.round(v * 128.0), -127, 127).to(torch.int8)
            chunks.append(q.reshape(-1).view(torch.uint8))
        else:
            if noise:
                s = NOISE_SIGMA / math.sqrt(2.0)
                re += s * torch.randn(nb, n, generator=g, device=dev, dtype=torch.float64)
                im += s * torch.randn(nb, n, generator=g, device=dev, dtype=torch.float64)
            if fmt == "int8_iq":
                qr = torch.clamp(torch.round(re * 128.0), -127, 127).to(torch.int8)
                qi = torch.clamp(torch.round(im * 128.0), -127, 127).to(torch.int8)
                chunks.append(torch.stack([qr, qi], -1).reshape(-1).view(torch.uint8))
            elif fmt == "int16_iq":
                qr = torch.clamp(torch.round(re * 32768.0), -32767, 32767).to(torch.int16)
                qi = torch.clamp(torch.round(im * 32768.0), -32767, 32767).to(torch.int16)
                chunks.append(torch.stack([qr, qi], -1).reshape(-1).view(torch.uint8))
            else:
                raise ValueError("fmt must be int8_iq, int16_iq or int8_real_if")
    return torch.cat(chunks)


def truth_channel_start(sv: Sv, fs: float):
    """(code boundary sample, Doppler) of the received code period at t=0:
    the acquisition hit run_closed_loop derives (test_tracking.cpp:378-384)."""
    boundary = int(round(sv.delay_chips / CHIP_RATE * fs))
    return boundary, sv.doppler_hz


def synth_gpu(ctx, n_ms: int, fs: float, recordings, *, fmt: str = "int16_iq", if_hz: float = 0.0,
              seed: int = 1, noise: bool = True, ms0: int = 0, out=None):
    """Many recordings at once on the GPU (l1rxg_simulate, the CUDA
    restatement of SimStream's raw mode, simsource.hpp:194-413):
    `recordings` is a list of Sv lists (one per recording, the same length);
    returns (or fills) a torch uint8 tensor [n_rec, n_ms * n * bytes_per_sample]
    on the context's device.  Noise is Philox-counted by sample index, so
    chunked calls (ms0) give the same bytes as one call."""
    import ctypes as C

    import torch

    from . import abi
    from ._native import check
    fmts = {"int8_iq": (abi.FMT_INT8_IQ, 2), "int16_iq": (abi.FMT_INT16_IQ, 4),
            "int8_real_if": (abi.FMT_INT8_REAL_IF, 1)}
    f, bps = fmts[fmt]
    n = llround(fs / 1000.0)
    n_rec = len(recordings)
    n_sv = len(recordings[0]) if n_rec else 0
    arr = (abi.SimSv * max(1, n_rec * n_sv))()
    for r, svs in enumerate(recordings):
        if len(svs) != n_sv:
            raise ValueError("every recording needs the same number of satellites")
        for k, sv in enumerate(svs):
            arr[r * n_sv + k] = abi.SimSv(sv.delay_chips, sv.doppler_hz, sv.doppler_rate, sv.phase0,
                                          sv.cn0_dbhz, sv.prn, 0)
    nbytes = n_ms * n * bps
    if out is None:
        out = torch.empty((n_rec, nbytes), dtype=torch.uint8, device=f"cuda:{ctx.device}")
    check(ctx._lib.l1rxg_simulate(ctx.handle, C.cast(arr, C.c_void_p), n_sv, n_rec, C.c_double(fs),
                                 C.c_double(if_hz), f, C.c_int64(ms0), n_ms, C.c_uint64(seed & (2**64 - 1)),
                                 1 if noise else 0, C.c_void_p(out.data_ptr()), C.c_int64(out.stride(0))))
    return out
