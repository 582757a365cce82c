#!/usr/bin/env python
"""bench.py -- tracking-correlator throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gpu|reference]
                    [--config 2|1|3|4]

Metric (BASELINE.json): correlator throughput in G sample-taps/s (one input
sample x one code tap, I and Q), and the real-time channel count per B200
(channel-epochs/s / 1000, the analogue of capacity = 1e6/avg_ns,
bench.hpp:26-30).

Workload at N=1 (BASELINE.json configs[1], "config 2"): 12 channels, PRNs
1-12, one shared int8 real-IF stream at 16.368 MHz with a 4.092 MHz IF,
Doppler U(+-5 kHz), code phase U[0,1023), C/N0 U[35,50] dB-Hz + AWGN,
E/P/L at 0.5 chip, 10000 1-ms blocks, PLL/DLL/FLL closed on device.
A step = ingest (mixer + half-band FIR) of the whole recording + closed-loop
tracking of every channel over every block.  Synthetic seeded data
(paper_1907_00463_b200/simsource.py); loops start from truth
(test_tracking.cpp:378-384) with lock_fail_limit = INT_MAX so every channel
computes every epoch.

value: device time (CUDA events on the library's stream) with the raw bytes
already resident in HBM.  e2e: the same step through the public API from
pinned host memory -- chunked H2D + ingest + tracking, then the epoch
records read back to the host -- all inside the timed region.
Multi-GPU: one process per GPU, each rank tracks its own seeded recording
(weak scaling, no collective on the data path); max over ranks; the epoch
records are gathered to rank 0 over NCCL after the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "correlator throughput (G sample-taps/s) and real-time channel count per B200"
UNIT = "G sample-taps/s"

CONFIGS = {
    # name: (fmt, fs, if_hz, n_channels, taps kind, blocks, seed)
    1: dict(fmt="int8_real_if", fs=16.368e6, if_hz=4.092e6, channels=1, taps="epl", blocks=1000, seed=1,
            desc="config1: PRN 1, int8 real IF 16.368 MHz / 4.092 MHz IF, +1.2 kHz, 45 dB-Hz, E/P/L, 1000 blocks"),
    2: dict(fmt="int8_real_if", fs=16.368e6, if_hz=4.092e6, channels=12, taps="epl", blocks=10000, seed=2,
            desc="config2: 12 channels PRN 1-12 on one int8 real-IF stream, 16.368 MHz / 4.092 MHz IF, "
                 "E/P/L 0.5 chip, 10000 1-ms blocks, closed loop"),
    3: dict(fmt="int16_iq", fs=16.368e6, if_hz=0.0, channels=32, taps="monitor", blocks=10000, seed=3,
            desc="config3: 32 channels x 11 taps (0.1 chip over +-0.5) + 2 loop taps, complex int16 at "
                 "16.368 MHz, 8 authentic + 8 spoofed PRNs, 10000 blocks"),
    4: dict(fmt="int16_iq", fs=65.472e6, if_hz=0.0, channels=12, taps="wide7", blocks=1000, seed=1000,
            desc="config4 (one recording per GPU-rank slice): 12 channels x 7 taps (0.25 chip), complex "
                 "int16 at 65.472 MHz, 1000 blocks"),
}


def make_taps(kind):
    from paper_1907_00463_b200 import abi
    if kind == "epl":
        return abi.Taps.epl(0.5)
    if kind == "monitor":
        return abi.Taps.make([round(-0.5 + 0.1 * k, 10) for k in range(11)] + [0.25, -0.25],
                             early=11, prompt=5, late=12, n_counted=11)
    return abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)


def scenario(cfg_id, seed):
    """Satellites and channel hand-offs of a config (seeded)."""
    from paper_1907_00463_b200 import simsource as ss
    c = CONFIGS[cfg_id]
    rng = np.random.default_rng(seed)
    if cfg_id == 1:
        svs = [ss.Sv(prn=1, cn0_dbhz=45.0, doppler_hz=1200.0, delay_chips=rng.uniform(0, 1023))]
        chans = [(svs[0], 1)]
    elif cfg_id == 2:
        svs = [ss.Sv(prn=p, cn0_dbhz=rng.uniform(35, 50), doppler_hz=rng.uniform(-5000, 5000),
                     delay_chips=rng.uniform(0, 1023)) for p in range(1, 13)]
        chans = [(sv, sv.prn) for sv in svs]
    elif cfg_id == 3:
        auth = [ss.Sv(prn=p, cn0_dbhz=rng.uniform(38, 48), doppler_hz=rng.uniform(-5000, 5000),
                      delay_chips=rng.uniform(0, 1000)) for p in (1, 3, 6, 9, 12, 17, 22, 28)]
        spoof = [ss.Sv(prn=a.prn, cn0_dbhz=a.cn0_dbhz + 3.0, doppler_hz=a.doppler_hz,
                       delay_chips=a.delay_chips + rng.uniform(0.2, 0.6)) for a in auth]
        svs = auth + spoof
        chans = [(a, a.prn) for a in auth for _ in range(4)]  # 4 monitor channels per PRN
    else:
        nvis = int(rng.integers(8, 13))
        prns = rng.choice(np.arange(1, 33), 12, replace=False)
        svs = [ss.Sv(prn=int(p), cn0_dbhz=rng.uniform(30, 50), doppler_hz=rng.uniform(-5000, 5000),
                     delay_chips=rng.uniform(0, 1023)) for p in prns[:nvis]]
        absent = [ss.Sv(prn=int(p), cn0_dbhz=30.0, doppler_hz=rng.uniform(-5000, 5000),
                        delay_chips=rng.uniform(0, 1023)) for p in prns[nvis:]]
        chans = [(sv, sv.prn) for sv in svs + absent]
    return c, svs, chans


def stream_manifest(raw_row, seed, svs, fmt):
    """Manifest of a synthetic stream: seed, signal parameters and
    the SHA-256 of its raw bytes (the CPU checker consumes the same bytes)."""
    import hashlib
    h = hashlib.sha256(raw_row.cpu().numpy().tobytes()).hexdigest()
    return {"seed": int(seed), "fmt": fmt, "bytes": int(raw_row.numel()), "sha256": h,
            "svs": [{"prn": sv.prn, "cn0_dbhz": round(sv.cn0_dbhz, 3), "doppler_hz": round(sv.doppler_hz, 3),
                     "delay_chips": round(sv.delay_chips, 4)} for sv in svs]}


def synth_config4(ctx, seed0, n_rec, blocks, fs, out=None):
    """Config-4 recordings seed0 .. seed0 + n_rec - 1 on the GPU in one call
    (l1rxg_simulate, the CUDA SimStream restatement): recording j's visible
    SVs (scenario(4, seed0 + j)) padded to 12 with silent entries; noise keyed
    by (seed0, j)."""
    from paper_1907_00463_b200 import simsource as ss
    rows = []
    for j in range(n_rec):
        _, svs, _ = scenario(4, seed0 + j)
        rows.append(svs + [ss.Sv(prn=1, cn0_dbhz=-200.0)] * (12 - len(svs)))
    return ss.synth_gpu(ctx, blocks, fs, rows, fmt="int16_iq", seed=seed0, out=out)


def channel_inits(chans, fs, lock_fail_limit_inf=True):
    from paper_1907_00463_b200 import simsource as ss
    from paper_1907_00463_b200.tracking import init_channel_from_acquisition
    out = []
    for sv, prn in chans:
        b, d = ss.truth_channel_start(sv, fs)
        out.append(init_channel_from_acquisition(prn, d, 0, b, 0, fs))
    return out


class ClockSampler:
    """nvidia-smi-equivalent NVML sampling of SM clock and throttle reasons
    during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def fp32_peak_tflops(sm_mhz):
    # 148 SMs x 128 FP32 lanes x 2 flop (FMA) at the SM clock -- the FP32
    # pipe issue roof (not in MEASURED_PEAKS.json, which has HBM and bf16)
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


def ops_per_sample_tap(T, C, real_if):
    # FP32-pipe instructions per sample-tap (FMA = 1) of the
    # direct algorithm: I/Q MAC 2 + carrier wipe 4/T + IF FIR F/(C T)
    return 2.0 + 4.0 / T + (13.0 / (C * T) if real_if else 0.0)


def cpu_reference_run(raw_np, c, inits, cfg_struct, blocks, threads):
    """The reference's own receiver tracking path on host cores
    (oracle/_ref: SampleSource producer + track_epoch pool, batched kernel)."""
    import ctypes as C
    import oracle
    from paper_1907_00463_b200 import abi
    n = int(round(c["fs"] / 1000))
    fmt = {"int8_real_if": abi.FMT_INT8_REAL_IF, "int16_iq": abi.FMT_INT16_IQ,
           "int8_iq": abi.FMT_INT8_IQ}[c["fmt"]]
    bps = abi.BYTES_PER_SAMPLE[fmt]
    with tempfile.NamedTemporaryFile(suffix=".bin", delete=False, dir="/dev/shm" if os.path.isdir("/dev/shm") else None) as f:
        f.write(raw_np[: blocks * n * bps].tobytes())
        path = f.name
    try:
        arr = (abi.Channel * len(inits))(*inits)
        wall, trk = C.c_double(), C.c_double()
        ce = C.c_int64()
        rc = oracle.ref().ref_bench_pipeline(path.encode(), fmt, c["fs"], c["if_hz"], len(inits), arr,
                                             C.byref(cfg_struct), abi.KERNEL_BATCHED, threads,
                                             blocks, C.byref(wall), C.byref(trk), C.byref(ce), None)
        if rc:
            raise RuntimeError(oracle.ref().ref_last_error().decode())
    finally:
        os.unlink(path)
    return wall.value, trk.value, ce.value


def cpu_port_run(x_cplx, inits, cfg_struct, taps, fs, blocks, threads, chan_stream=None):
    """Builder K-tap restatement (oracle port) for multi-tap configs.
    `x_cplx` is one complex stream or a list of them (`chan_stream` binds
    each channel to its stream)."""
    import oracle
    n = int(round(fs / 1000))
    xs = x_cplx if isinstance(x_cplx, list) else [x_cplx]
    cs = chan_stream if chan_stream is not None else [0] * len(inits)
    t = time.perf_counter()
    _, done, _, _ = oracle.track_run(inits, cs, xs, n, cfg_struct, taps, fs,
                                     blocks, threads=threads, records=False)
    return time.perf_counter() - t, int(sum(done))


GRID = dict(fs=16.368e6, if_hz=4.092e6, n_prns=32, bins=np.arange(-10000.0, 10000.1, 500.0),
            blocks=20, seed=5,
            desc="config5: search grid, PRNs 1-32 x 41 Doppler bins (+-10 kHz / 500 Hz) x 2046 "
                 "half-chip delays, 20 x 1-ms int8 real-IF blocks at 16.368 MHz / 4.092 MHz IF, "
                 "noncoherent |I+jQ| accumulation, 6 SVs at C/N0 U[25,45]")


def run_grid(args, rank, world, local, dist):
    """Config 5: the correlator-bank search grid over one recording, its 32
    PRNs sharded over the ranks (strong scaling: shard_list of PRNs 1-32),
    every rank's plane gathered to rank 0 over NCCL inside the e2e leg."""
    import torch
    from paper_1907_00463_b200 import abi, simsource as ss
    from paper_1907_00463_b200.shard import shard_list
    g = GRID
    rng = np.random.default_rng(g["seed"])
    prns_sv = rng.choice(np.arange(1, 33), 6, replace=False)
    svs = [ss.Sv(prn=int(p), cn0_dbhz=rng.uniform(25, 45), doppler_hz=rng.uniform(-9000, 9000),
                 delay_chips=rng.uniform(0, 1023)) for p in prns_sv]
    fs, N, blocks = g["fs"], 16368, g["blocks"]
    all_prns = np.arange(1, 33, dtype=np.int32)
    prns = np.array(shard_list(list(all_prns), world, rank), dtype=np.int32)
    bins = g["bins"]
    direct_st = float(all_prns.size) * bins.size * 2046 * N * blocks  # direct-equivalent sample-taps, all ranks
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    raw = ss.synth(blocks, fs, svs, fmt="int8_real_if", if_hz=g["if_hz"], seed=g["seed"], device=dev)
    if args.impl == "reference":
        if rank != 0:
            return
        import oracle
        x = oracle.ingest(raw.cpu().numpy(), abi.FMT_INT8_REAL_IF, fs, g["if_hz"])
        walls, kind = [], "port"
        if oracle.acq_available() and torch.cuda.is_available():
            # the reference's own acquire_pcs (acquisition.hpp:189-222; FFTW's
            # API served by cuFFTW): 2 PRNs x 41 bins x 20 blocks per step,
            # scaled per direct-equivalent cell
            kind = "reference"
            for step in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                for p in (int(prns_sv[0]), 7):
                    oracle.ref_acquire_pcs(x, p, fs, -10000, 10000, 500, blocks)
                if step >= args.warmup:
                    walls.append(time.perf_counter() - t0)
            st = 2 * bins.size * 2046 * N * blocks * 1.0
            sample = ("2 PRNs x 41 bins x 20 blocks: the reference's acquire_pcs (FFT circular correlation, "
                      "acquisition.hpp:189-222) with FFTW's API served by cuFFTW (FFTW3 absent)")
        else:
            # bounded sample of the direct restatement: 2 PRNs x 4 bins x 1 block
            for step in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                for p in (int(prns_sv[0]), 7):
                    oracle.search_grid(x[:N], N, 1, p, fs, bins[18:22], 8, 2046)
                if step >= args.warmup:
                    walls.append(time.perf_counter() - t0)
            st = 2 * 4 * 2046 * N * 1.0
            sample = "2 PRNs x 4 bins x 1 block, direct time-domain restatement of acquire_pcs"
        v = st / statistics.mean(walls) / 1e9
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": statistics.mean(walls) * 1e3, "higher_is_better": True,
                          "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": g["desc"]},
                          "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": kind, "sample": sample},
                          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    from paper_1907_00463_b200.tracking import Context, search_grid, search_grid_timing
    ctx = Context(local)
    nbytes = raw.numel()
    for _ in range(args.warmup):
        search_grid(ctx, nbytes, abi.FMT_INT8_REAL_IF, fs, g["if_hz"], blocks, prns, bins,
                    device_ptr=raw.data_ptr())
    clocks = ClockSampler(local)
    fold_ms = corr_ms = 0.0
    if dist:
        dist.barrier()
    with clocks:
        for _ in range(args.steps):
            plane = search_grid(ctx, nbytes, abi.FMT_INT8_REAL_IF, fs, g["if_hz"], blocks, prns,
                                bins, device_ptr=raw.data_ptr())
            a, b = search_grid_timing(ctx)
            fold_ms += a
            corr_ms += b
    dev_ms = (fold_ms + corr_ms) / args.steps
    t_max = dev_ms
    if dist:
        tt = torch.tensor([dev_ms], device=torch.device("cuda", local))
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())

    # e2e: host bytes in (pinned), this rank's PRN planes out as float32 --
    # into pinned host memory at N = 1; into device memory, gathered to rank
    # 0 over NCCL and read back there, at N > 1
    host = ctx.host_alloc(nbytes)
    host[:] = raw.cpu().numpy()
    plane_bytes = prns.size * bins.size * 2046 * 4
    out_host = ctx.host_alloc(all_prns.size * bins.size * 2046 * 4).view(np.float32)
    out_dev = torch.empty(plane_bytes, dtype=torch.uint8, device=torch.device("cuda", local)) if dist else None

    def step_e2e():
        if not dist:
            return search_grid(ctx, host, abi.FMT_INT8_REAL_IF, fs, g["if_hz"], blocks, prns, bins, out=out_host,
                               dtype=np.float32)
        from paper_1907_00463_b200.shard import gather_bytes
        search_grid(ctx, host, abi.FMT_INT8_REAL_IF, fs, g["if_hz"], blocks, prns, bins,
                    out_device_ptr=out_dev.data_ptr(), dtype=np.float32)
        outs = gather_bytes(out_dev, dist, dst=0)
        if rank != 0:
            return None
        allp = torch.cat(outs)
        torch.from_numpy(out_host.view(np.uint8)).copy_(allp)
        return out_host.reshape(all_prns.size, bins.size, 2046)
    step_e2e()
    if dist:
        dist.barrier()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        full = step_e2e()
    e2e_ms = (time.perf_counter() - w0) * 1e3 / args.steps
    if dist:
        tt = torch.tensor([e2e_ms], device=torch.device("cuda", local))
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    if rank != 0:
        dist.destroy_process_group()
        return
    # detections (acquisition.hpp:114-149) from the gathered full plane
    from paper_1907_00463_b200.tracking import pick_peak
    det = []
    for p in prns_sv:
        r = pick_peak(full[int(p) - 1], bins, fs, prn=int(p))
        det.append({"prn": int(p), "bin_hz": r.doppler_hz, "delay_chips": r.code_delay_chips,
                    "ratio": round(float(r.ratio), 2), "detected": bool(r.detected)})
    # untimed parity: the full plane against the reference's own acquire_pcs
    # plane (acquisition.hpp over cuFFTW) at three bins of three PRNs (two
    # present, one absent), within 1e-5 of the largest cell
    parity = None
    if not args.no_parity:
        try:
            import oracle
            if oracle.acq_available():
                t0p = time.perf_counter()
                x = oracle.ingest(raw.cpu().numpy(), abi.FMT_INT8_REAL_IF, fs, g["if_hz"])
                absent = next(p for p in range(1, 33) if p not in set(int(q) for q in prns_sv))
                worst = 0.0
                for sv_i, p in ((0, int(prns_sv[0])), (1, int(prns_sv[1])), (None, absent)):
                    k = int(np.argmin(np.abs(bins - svs[sv_i].doppler_hz))) if sv_i is not None else 20
                    sel = sorted({max(0, min(bins.size - 1, k + o)) for o in (-1, 0, 1)})
                    want = oracle.ref_pcs_plane(x, blocks, p, fs, bins[sel])[:, ::8]
                    worst = max(worst, float(np.abs(full[p - 1][sel] - want).max() / want.max()))
                parity = {"ok": worst <= 1e-5, "worst_cell": worst, "tolerance": 1e-5,
                          "sample": "3 bins x 3 PRNs (2 present, 1 absent) of the full 32-PRN plane",
                          "reference": "acquire_pcs plane, acquisition.hpp + fft.hpp over cuFFTW",
                          "seconds": round(time.perf_counter() - t0p, 1)}
        except Exception as ex:  # reported, not fatal
            parity = {"ok": None, "error": repr(ex)}
    clk = clocks.summary()
    sm_mhz = clk["sm_mhz"] or 1965.0
    path = os.environ.get("L1RXG_GRID", "mma")
    if os.environ.get("L1RXG_GRID_FP32", "0") not in ("", "0"):
        path = "fp32"
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    n_rows = 32 * ((blocks + 4) // 5)
    if path == "fp32":  # FP32-pipe circulant kernel: 2 FFMA x 2 flop per cell-chip
        corr_flops = float(prns.size) * bins.size * blocks * 2 * 1023 * 1023 * 4
        peak = fp32_peak_tflops(sm_mhz)
        bound, note = "fp32", ("executed algorithm: two 1023-point circulant +-1 correlations per "
                               "(PRN, bin, block) on the FP32 pipes; direct-equivalent rate in value")
        launches = 3
    elif path == "gemm":  # cuBLAS bf16x3 GEMM: M=1024 delays, N=2*2*bins*blocks rows, K=3*1024
        corr_flops = 2.0 * 1024 * (4 * bins.size * blocks) * 3072 * prns.size
        peak = peaks.get("bf16_tflops", 2250.0)
        bound, note = "tensor", ("executed algorithm: per PRN one bf16 GEMM (fp32 folds split into "
                                 "three bf16 terms, +-1 circulant code matrix, fp32 accumulate) via "
                                 "cuBLAS on tcgen05; peak = MEASURED_PEAKS bf16_tflops (burst); the "
                                 "corr time also holds the split, circulant-build and |.| kernels")
        launches = 6
    else:  # K4c: hand-written tcgen05 int8 GEMM, M=1024 delays x N=n_rows digit rows per group x K=1024
        corr_flops = 2.0 * 1024 * n_rows * (2 * bins.size) * 1024 * prns.size
        peak = 2.0 * peaks.get("bf16_tflops", 2250.0)
        bound, note = "tensor", ("executed algorithm: grid_mma_kernel, one tcgen05 kind::i8 GEMM (folds as "
                                 "three signed base-256 digits of 24-bit vector-quantised integers x the "
                                 "+-1 circulant generated on chip into TMEM, exact int32 accumulation in "
                                 "TMEM) with the digit recombination, |.| and the 20-block noncoherent sum "
                                 "fused into the epilogue; %d digit rows per (bin, parity) group; peak = "
                                 "2 x MEASURED_PEAKS bf16_tflops (B200 dense int8 rate = 2 x bf16; against "
                                 "the nominal 4.5 POPS the fraction is frac_vs_nominal); the corr time also "
                                 "holds the digit split and its memset" % n_rows)
        launches = 4
    achieved = corr_flops / (corr_ms / args.steps * 1e-3) / 1e12
    line = {"metric": METRIC, "value": direct_st / (t_max * 1e-3) / 1e9, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded; 6 SVs)",
            "config": {"workload": g["desc"], "delay_grid": "d = 8k samples, k < 2046",
                       "value_basis": "direct-equivalent sample-taps (PRN x bin x delay x sample)",
                       "parallelism": f"strong: 32 PRNs over {world} rank(s) ({prns.size} on rank 0), "
                                      f"planes gathered to rank 0 (NCCL) in the e2e leg"},
            "kernel_ms_per_step": {"ingest_fold": fold_ms / args.steps, "corr": corr_ms / args.steps},
            "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None, "note": note,
                         "frac_vs_nominal": (None if path == "fp32" else
                                             achieved / (4500.0 if path == "mma" else 2250.0))},
            "e2e": {"value": direct_st / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
                    "ms_per_step": e2e_ms, "h2d_bytes_per_step": int(nbytes) * world,
                    "d2h_bytes_per_step": int(full.size * 4)},
            "detections": det, "gpu_launches": launches * args.steps, "clocks": clk, "grid_path": path,
            "parity": parity}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


BATCH = dict(recordings=512, chunk_blocks=50, blocks_per_step=1000,
             desc="config4: 512 independent seeded recordings x 12 channels x 7 taps (0.25 chip), "
                  "complex int16 I/Q at 65.472 MHz, 8-12 visible SVs per recording, Doppler U(+-5 kHz), "
                  "C/N0 U[30,50] dB-Hz")


def batch_parity(trk, raw, recs, inits, cstream, n, fs, cfg, taps, n_rec=4, per_rec=2):
    """Untimed in-bench parity (oracle/replay.py): every epoch of `per_rec`
    channels (the first and the last: a visible SV and, when fewer than 12
    are visible, a noise-only channel) of each of the first `n_rec` local
    recordings, re-run by the CPU oracle from the GPU's own pre-state --
    sums within 1e-5 x max|E/P/L| and the 7 tap sums, NCO advance
    bit-exact, loop outputs within 1e-5."""
    from concurrent.futures import ThreadPoolExecutor
    import oracle
    from oracle.replay import replay_channel
    from paper_1907_00463_b200 import abi
    t0 = time.perf_counter()
    R = min(n_rec, len(recs))
    picks = []
    for j in range(R):
        chans = [c for c in range(len(inits)) if cstream[c] == j]
        picks += sorted({chans[0], chans[-1]})[:per_rec]
    xs = {j: oracle.ingest(raw[j].cpu().numpy(), abi.FMT_INT16_IQ, fs) for j in range(R)}
    got = {c: trk.records(c, tap_sums=True) for c in picks}

    def one(c):
        recs_c, ts = got[c]
        return replay_channel(oracle, inits[c], recs_c, xs[cstream[c]], n, cfg, taps, fs, tap_sums=ts)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        res = list(ex.map(one, picks))
    worst = {k: max(r[0][k] for r in res) for k in ("sums", "taps", "loop", "cn0")}
    n_bad = sum(r[1] for r in res)
    first = next((r[2] for r in res if r[2]), None)
    checked = int(sum(len(got[c][0]) for c in picks))
    ok = worst["sums"] <= 1e-5 and worst["taps"] <= 1e-5 and worst["loop"] <= 1e-5 and n_bad == 0
    return {"ok": bool(ok), "checked_channel_epochs": checked, "channels": picks,
            "recordings": list(range(R)), "worst_sum": worst["sums"], "worst_tap_sum": worst["taps"],
            "worst_loop": worst["loop"], "worst_cn0_rel": worst["cn0"], "exact_field_mismatches": n_bad,
            "first_mismatch": first, "tolerance": {"sums": 1e-5, "loop": 1e-5, "nco": "bit-exact"},
            "oracle": "oracle/l1rx_oracle.c track_epoch (tracking.hpp:520-618 restated; 3-tap instance "
                      "pinned to the reference build), replayed from the GPU's own pre-state",
            "seconds": round(time.perf_counter() - t0, 1)}


def host_budget(need_local, world):
    """Whether `need_local` bytes of pinned host memory per rank fit this host
    with every local rank asking the same (ranks share the host's RAM)."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        return False, 0
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    margin = 24 << 30  # the processes themselves, torch, page cache
    return need_local * local_world + margin <= avail, avail


def batch_e2e(ctx, raw, recs, inits, cstream, taps, cfg, fs, n, blocks, chunk_b, T, args, world, dist,
              dev, barrier):
    """e2e leg of config 4 through the public API: the local recordings
    live in pinned host memory as `blocks / chunk_b` chunk buffers
    [recording][chunk_b blocks]; each step resets a ring tracker, streams
    every chunk with l1rxg_tracker_push_strided (H2D on the library's copy
    stream into two alternating device staging blocks, overlapped with the
    previous chunk's tracking) + run, and reads every epoch record back
    into pinned host memory."""
    import torch
    from paper_1907_00463_b200 import abi
    from paper_1907_00463_b200.tracking import Tracker
    nrl = len(recs)
    cb = chunk_b * n * 4
    n_chunks = -(-blocks // chunk_b)
    need = nrl * blocks * n * 4
    fits, avail = host_budget(need, world)
    e2e_recs = nrl
    while not fits and e2e_recs > 1:  # never on the measured boxes (196 GB host, 134 GB input)
        e2e_recs //= 2
        fits, avail = host_budget(e2e_recs * blocks * n * 4, world)
    if not fits:
        return {"value": None, "unit": UNIT, "skipped": "host memory (%.0f GB available)" % (avail / 1e9)}
    t_fill = time.perf_counter()
    chunks = []
    for c in range(n_chunks):
        a, b = c * cb, min((c + 1) * cb, blocks * n * 4)
        buf = ctx.host_alloc(e2e_recs * (b - a)).reshape(e2e_recs, b - a)
        torch.from_numpy(buf).copy_(raw[:e2e_recs, a:b])  # one D2H per chunk (a device-side gather first)
        chunks.append(buf)
    torch.cuda.synchronize()
    t_fill = time.perf_counter() - t_fill
    nci = sum(1 for s_ in cstream if s_ < e2e_recs)
    te = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits[:nci], chan_stream=cstream[:nci],
                 n_streams=e2e_recs, taps=taps, cfg=cfg, ring_samples=(chunk_b + 4) * n,
                 max_records=blocks, cta_mode=abi.CTA_SEGMENT)
    rec_bytes = te.records_nbytes()
    rec_pinned = ctx.host_alloc(rec_bytes)  # the step's records land in pinned host memory

    def step_e2e():
        te.reset()
        for buf in chunks:
            te.push_strided(buf)
            te.run()
        te.records_raw(dst_ptr=rec_pinned.ctypes.data)
        te.sync()

    step_e2e()
    te.timing()
    barrier()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        step_e2e()
    e2e_ms = (time.perf_counter() - w0) * 1e3 / args.steps
    _, _, e2e_launches = te.timing()
    if dist:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_epochs_local = float(te.epoch_counts().sum())
    e2e_epochs = e2e_epochs_local
    if dist:  # every rank's channel-epochs of the step
        tt = torch.tensor([e2e_epochs_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        e2e_epochs = float(tt.item())
    out = {"value": e2e_epochs * n * T / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": int(e2e_recs * blocks * n * 4), "d2h_bytes_per_step": int(rec_bytes),
           "blocks_per_step": blocks, "recordings_per_rank": e2e_recs, "channel_epochs_per_rank": e2e_epochs_local,
           "h2d_gbs": e2e_recs * blocks * n * 4 / (e2e_ms * 1e-3) / 1e9,
           "gpu_launches_per_step": e2e_launches / max(1, args.steps),
           "pinned_source": "%d chunk buffers of %d blocks x %d recordings (%.1f GB each, %.1f GB pinned; "
                            "filled in %.1f s, untimed)" % (n_chunks, chunk_b, e2e_recs, e2e_recs * cb / 1e9,
                                                           e2e_recs * blocks * n * 4 / 1e9, t_fill),
           "path": "pinned host chunk [recording][%d blocks] -> l1rxg_tracker_push_strided (H2D on the copy "
                   "stream into one of two device staging blocks + one raw-ring copy launch) -> "
                   "l1rxg_tracker_run (segment correlator over the chunk) -> ... -> records_raw to pinned "
                   "host; wall clock per step, max over ranks" % chunk_b}
    del te
    del chunks
    return out


def run_batch(args, rank, world, local, dist, emit=True):
    """Config 4: many independent recordings, sharded by recording over the
    ranks (strong scaling: the 512 recordings are split, no data-path
    collective).  One step = every local recording x `blocks_per_step`
    1-ms blocks from the acquisition hand-off: lock-step strided pushes of
    `chunk_blocks` (one decode launch for all recordings) + one tracking
    launch per chunk with two narrow CTAs per SM."""
    import torch
    from paper_1907_00463_b200 import abi, simsource as ss
    from paper_1907_00463_b200.shard import shard_range
    from paper_1907_00463_b200.tracking import Context, Tracker
    c = CONFIGS[4]
    fs, n = c["fs"], int(round(c["fs"] / 1000))
    blocks = args.blocks or BATCH["blocks_per_step"]
    chunk_b = min(BATCH["chunk_blocks"], blocks)
    n_rec_total = args.recordings or BATCH["recordings"]
    recs = shard_range(n_rec_total, world, rank)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    # The whole workload (every recording x every block) is resident in HBM:
    # raw cint16 + the per-recording float2 ring + records/tap sums.  If the
    # device cannot hold it, the step shrinks to the largest chunk multiple
    # that fits and config.blocks_per_step says so.
    want_blocks = blocks
    free = torch.cuda.mem_get_info(dev)[0]
    per_block = len(recs) * (n * 4 + 12 * (248 + 2 * 8 * 8))
    fixed = len(recs) * (chunk_b + 5) * n * 8 + (6 << 30)
    if fixed + per_block * blocks > free:
        blocks = max(chunk_b, (free - fixed) // per_block // chunk_b * chunk_b)
    taps = make_taps("wide7")
    cfg = abi.TrackingCfg.default()
    cfg.lock_fail_limit = 2**31 - 1
    T = taps.n_counted
    inits, cstream = [], []
    bytes_rec = blocks * n * 4
    raw = torch.empty((len(recs), bytes_rec), dtype=torch.uint8, device=dev)
    ctx = Context(local)
    t_syn = time.perf_counter()
    if len(recs):  # recs are consecutive: one simulator call for this rank's recordings
        synth_config4(ctx, c["seed"] + recs[0], len(recs), blocks, fs, out=raw)
    for j, r in enumerate(recs):
        _, svs, chans = scenario(4, c["seed"] + r)
        ci = channel_inits(chans, fs)
        inits += ci
        cstream += [j] * len(ci)
    torch.cuda.synchronize()
    t_syn = time.perf_counter() - t_syn
    C_ch = len(inits)
    manifest0 = stream_manifest(raw[0], c["seed"] + recs[0], scenario(4, c["seed"] + recs[0])[1],
                                "int16_iq") if len(recs) else None
    if manifest0:
        manifest0["generator"] = ("l1rxg_simulate (CUDA SimStream raw mode), Philox noise keyed by "
                                  "(seed %d, recording index)" % (c["seed"] + recs[0]))
    trk = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, chan_stream=cstream, n_streams=len(recs),
                  taps=taps, cfg=cfg, ring_samples=(chunk_b + 4) * n, max_records=blocks,
                  cta_mode={"segment": abi.CTA_SEGMENT, "throughput": abi.CTA_THROUGHPUT,
                            "latency": abi.CTA_LATENCY}[args.cta],
                  ring_raw=args.ring_raw)
    stream = torch.cuda.ExternalStream(trk.cuda_stream(), device=dev)
    chunk = chunk_b * n * 4

    attached = args.cta == "segment"
    if attached:  # the resident recordings are the rings: no ingest pass, one launch per step
        trk.attach_device(raw.data_ptr(), bytes_rec // 4, bytes_rec)

    def step_device():
        trk.reset()
        if attached:
            trk.run()
            return
        for o in range(0, bytes_rec, chunk):
            trk.push_device_strided(raw.data_ptr() + o, min(chunk, bytes_rec - o), bytes_rec)
            trk.run()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step_device()
    trk.sync()
    trk.timing()
    clocks = ClockSampler(local)
    barrier()
    with clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step_device()
        e1.record(stream)
        e1.synchronize()
    barrier()
    dev_ms = e0.elapsed_time(e1)
    ingest_ms, track_ms, launches = trk.timing()
    t_max = dev_ms
    if dist:
        tt = torch.tensor([dev_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    ms_per_step = t_max / args.steps
    counts = trk.epoch_counts()
    assert int(counts.min()) >= blocks - 2, counts.min()
    epochs_local = float(counts.sum())
    tot = torch.tensor([epochs_local], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    epochs_all = float(tot.item())
    sample_taps_all = epochs_all * n * T
    value = sample_taps_all / (ms_per_step * 1e-3) / 1e9

    # ---- end-of-run gather of the records to rank 0, untimed
    gathered = None
    if dist:
        from paper_1907_00463_b200.shard import gather_bytes
        rec_t = torch.empty(trk.records_nbytes(), dtype=torch.uint8, device=dev)
        trk.records_raw(dst_ptr=rec_t.data_ptr(), device=True)
        outs = gather_bytes(rec_t, dist, dst=0)
        gathered = sum(int(o.numel()) for o in outs) if rank == 0 else None
        del rec_t, outs

    # ---- untimed parity: oracle replay of a deterministic sample of epochs
    parity = None
    if rank == 0 and not args.no_parity:
        parity = batch_parity(trk, raw, recs, inits, cstream, n, fs, cfg, taps)

    # ---- e2e: the same step from pinned host memory, every block of every
    # local recording (bounded pinned chunks of chunk_b blocks, streamed
    # through l1rxg_tracker_push_strided into a ring tracker)
    e2e = None
    if not args.no_e2e:
        e2e = batch_e2e(ctx, raw, recs, inits, cstream, taps, cfg, fs, n, blocks, chunk_b, T, args,
                        world, dist, dev, barrier)
    if rank != 0:
        if emit:
            dist.destroy_process_group()
        return None
    clk = clocks.summary()
    sm_mhz = clk["sm_mhz"] or 1965.0
    track_launch_ms = track_ms / args.steps
    alg_flops = epochs_local * n * T * 2.0 * ops_per_sample_tap(T, 12, False)
    achieved = alg_flops / (track_launch_ms * 1e-3) / 1e12
    peak = fp32_peak_tflops(sm_mhz)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic_config4.json" if attached else "ncu_traffic_config4_trackkernel.json")
    launches_per_step = 1 if attached else -(-blocks // chunk_b)
    if os.path.exists(prof):  # measured DRAM bytes per channel-epoch x channel-epochs per launch
        per = json.load(open(prof)).get("dram_bytes_per_channel_epoch")
        traffic = per * epochs_local / launches_per_step if per else None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        threads = os.cpu_count() or 1
        cb = min(args.cpu_blocks, blocks, 1000)
        R = min(8, len(recs))  # >= 8 recordings x 1000 blocks, scaled linearly
        t_ing = time.perf_counter()
        xs = [oracle.ingest(raw[j, : cb * n * 4].cpu().numpy(), abi.FMT_INT16_IQ, fs) for j in range(R)]
        t_ing = time.perf_counter() - t_ing
        nci = sum(1 for s_ in cstream if s_ < R)
        wall, ce = cpu_port_run(xs, inits[:nci], cfg, taps, fs, cb, threads, chan_stream=cstream[:nci])
        del xs
        cpu = {"value": float(ce) * n * T / wall / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
               "scope": "tracking stage only (correlator + loop update, bench.hpp:59-102); ingest "
                        "(cint16 decode) timed separately",
               "tracking_s": wall, "ingest_s": t_ing,
               "sample": f"recordings 0-{R - 1}: {nci} channels x {cb} blocks (oracle K-tap "
                         f"restatement -- the reference has no 7-tap correlator -- on a {threads}-thread "
                         f"channel pool, {wall:.2f} s)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded per recording, paper_1907_00463_b200/simsource.py; loops start from truth)",
        "config": {"workload": BATCH["desc"], "recordings": n_rec_total, "channels": C_ch * world,
                   "taps_counted": T, "samples_per_block": n, "blocks_per_step": blocks,
                   "blocks_requested": want_blocks,
                   "chunk_blocks": None if attached else chunk_b, "cta_mode": args.cta,
                   "ingest": ("recordings attached in place (l1rxg_tracker_attach_device): the segment "
                              "correlator reads the resident cint16 by TMA, no ingest pass" if attached else
                              "strided device pushes (decode or raw copy into the rings) per chunk"),
                   "parallelism": f"strong: {n_rec_total} recordings over {world} rank(s)",
                   "l2": "inputs larger than L2 (raw %.1f GB + baseband ring %.1f GB per rank)" % (
                       raw.numel() / 1e9, len(recs) * (chunk_b + 5) * n * 8 / 1e9),
                   "synth_s": round(t_syn, 1),
                   "manifest_recording0": manifest0,
                   "lock_fail_limit": "INT_MAX (every channel computes every epoch)"},
        "realtime_channels": epochs_all / (ms_per_step * 1e-3) / 1000.0,
        "kernel_ms_per_step": {"ingest": ingest_ms / args.steps, "track": track_launch_ms},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_note": ("DRAM bytes per track_seg_kernel launch (all %d blocks of every "
                                      "recording), profiles/ncu_traffic_config4.json" % blocks) if attached
                                     else ("DRAM bytes per track_kernel launch (one %d-block chunk of every "
                                           "recording), profiles/ncu_traffic_config4_trackkernel.json" % chunk_b),
                     "peak_source": "148 SMs x 128 FP32 lanes x 2 x median SM clock under load "
                                    "(%.0f MHz); FP32 pipe roof per SURVEY 8d" % sm_mhz,
                     "alg_ops_per_sample_tap": ops_per_sample_tap(T, 12, False),
                     "hbm": {"achieved_gbs": (len(recs) * blocks * n * (4 if attached else 8))
                                             / (track_launch_ms * 1e-3) / 1e9,
                             "peak_gbs": peaks.get("hbm_gbs", 6450.0),
                             "note": ("unique cint16 bytes per step (each recording read in place once; its "
                                      "12 channels share it through L2)") if attached else
                                     ("unique float2 baseband bytes per step (each recording's ring read "
                                      "once; its 12 channels share it through L2)")}},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        "parity": parity,
    }
    if gathered is not None:
        line["records_gathered_bytes"] = gathered
    if not emit:
        return line
    if args.companion and world == 1:
        trk.close()
        del raw
        torch.cuda.empty_cache()
        line["companion_latency"] = companion_latency(args, local)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return line


def run_batch_reference(args, rank):
    """`--impl reference` for config 4: the reference's K-tap tracking path
    (oracle port: the reference's builder has no multi-tap batch driver to
    compile standalone) on every host thread, over a bounded sample of the
    workload — the first 8 recordings x 1000 blocks per step,
    same scenarios and seeds as the GPU arm."""
    import torch
    from paper_1907_00463_b200 import abi, simsource as ss
    import oracle
    if rank != 0:
        return None
    c = CONFIGS[4]
    fs, n = c["fs"], int(round(c["fs"] / 1000))
    per_step = min(args.blocks or 1000, 1000)
    R = 8
    taps = make_taps("wide7")
    cfg = abi.TrackingCfg.default()
    cfg.lock_fail_limit = 2**31 - 1
    T = taps.n_counted
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    xs, inits, cstream = [], [], []
    from paper_1907_00463_b200.tracking import Context
    raws = synth_config4(Context(0), c["seed"], R, per_step, fs).cpu().numpy()  # the device arm's rank-0 bytes
    for r in range(R):
        _, svs, chans = scenario(4, c["seed"] + r)
        xs.append(oracle.ingest(raws[r], abi.FMT_INT16_IQ, fs))
        ci = channel_inits(chans, fs)
        inits += ci
        cstream += [r] * len(ci)
    threads = os.cpu_count() or 1
    walls, ces = [], []
    for step in range(args.warmup + args.steps):
        # tracking stage only (bench.hpp:59-102); the cint16 decode ran above
        wall, ce = cpu_port_run(xs, inits, cfg, taps, fs, per_step, threads, chan_stream=cstream)
        if step >= args.warmup:
            walls.append(wall)
            ces.append(ce)
    w = statistics.mean(walls)
    v = statistics.mean(ces) * n * T / w / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": w * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": BATCH["desc"], "sample_recordings": R,
                                            "sample_blocks_per_step": per_step,
                                            "parallelism": f"{threads} host threads"},
            "realtime_channels": statistics.mean(ces) / w / 1000.0,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "scope": "tracking stage only (correlator + loop update, bench.hpp:59-102)",
                             "sample": f"{R} recordings ({len(inits)} channels) x {per_step} blocks per step "
                                       f"(oracle K-tap restatement: the reference has no 7-tap correlator; "
                                       f"its 3-tap instance equals the reference's scalar kernel)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return line


def companion_latency(args, local):
    """The latency view next to the throughput headline: config 2 (12
    channels on one int8 real-IF stream, 10 000 strictly sequential 1-ms
    epochs, the overlapped latency kernel), its value, e2e, per-epoch
    critical path and roofline fraction; `bench.py --config 2` gives the
    full line with its CPU baseline."""
    import copy
    import torch
    a = copy.copy(args)
    a.blocks, a.steps, a.warmup = 0, 3, 3
    a.no_cpu_baseline = True
    a.no_parity = True
    try:
        torch.cuda.empty_cache()
        ln = run_stream(a, 2, 0, 1, local, None, emit=False)
        torch.cuda.empty_cache()
        return {"workload": CONFIGS[2]["desc"], "value": ln["value"], "unit": ln["unit"],
                "ms_per_step": ln["ms_per_step"], "epoch_latency_us": ln["epoch_latency_us"],
                "realtime_channels": ln["realtime_channels"], "e2e": ln["e2e"], "roofline": ln["roofline"],
                "gpu_launches": ln["gpu_launches"], "clocks": ln["clocks"]}
    except Exception as ex:  # reported, never fatal for the headline line
        return {"error": repr(ex)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (default 4: the largest single-GPU workload)")
    ap.add_argument("--blocks", type=int, default=0, help="override the config's block count")
    ap.add_argument("--cpu-blocks", type=int, default=3000, help="CPU baseline sample (blocks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="config 4: skip the host-memory e2e leg")
    ap.add_argument("--no-parity", action="store_true", help="config 4: skip the untimed oracle replay")
    ap.add_argument("--e2e-chunk-ms", type=int, default=1000)
    ap.add_argument("--recordings", type=int, default=0, help="config 4: override 512 recordings")
    ap.add_argument("--cta", default="segment", choices=["segment", "throughput", "latency"],
                    help="config 4 CTA shape: segment correlator (raw cint16 ring), throughput, latency")
    ap.add_argument("--ring-raw", action="store_true", help="config 4: keep cint16 raw in the rings")
    ap.add_argument("--no-companion", dest="companion", action="store_false",
                    help="config 4: skip the config-2 latency companion measurement")
    args = ap.parse_args()

    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if args.impl == "reference":  # CPU arm: rank 0 alone runs and prints it
        if rank != 0:
            return None
        if args.config == 5:
            return run_grid(args, 0, 1, local, None)
        if args.config == 4:
            return run_batch_reference(args, 0)
        return run_stream(args, args.config, 0, 1, local, None)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.config == 5:
        return run_grid(args, rank, world, local, dist)
    if args.config == 4:
        return run_batch(args, rank, world, local, dist)
    return run_stream(args, args.config, rank, world, local, dist)


def stream_parity(trk, raw, inits, fmt, if_hz, n, fs, cfg, taps, every=25, head=200):
    """Untimed in-bench parity for configs 1-3 (oracle/replay.py): every
    `every`-th epoch of every channel plus the first `head` epochs of channel
    0, re-run by the CPU oracle from the GPU's own pre-state (sums 1e-5 x
    max|E/P/L| and every tap, NCO advance bit-exact, loop outputs 1e-5)."""
    import oracle
    from oracle.replay import replay_channel
    from concurrent.futures import ThreadPoolExecutor
    t0 = time.perf_counter()
    x = oracle.ingest(raw.cpu().numpy(), fmt, fs, if_hz)
    got = {c: trk.records(c, tap_sums=True) for c in range(len(inits))}

    def one(c):
        recs, ts = got[c]
        ks = sorted(set(range(0, len(recs), every)) | (set(range(min(head, len(recs)))) if c == 0 else set()))
        return replay_channel(oracle, inits[c], recs, x, n, cfg, taps, fs, tap_sums=ts, epochs=ks) + (len(ks),)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        res = list(ex.map(one, range(len(inits))))
    worst = {k: max(r[0][k] for r in res) for k in ("sums", "taps", "loop", "cn0")}
    n_bad = sum(r[1] for r in res)
    ok = worst["sums"] <= 1e-5 and worst["taps"] <= 1e-5 and worst["loop"] <= 1e-5 and n_bad == 0
    return {"ok": bool(ok), "checked_channel_epochs": int(sum(r[3] for r in res)),
            "sample": f"every {every}th epoch of every channel + epochs 0-{head - 1} of channel 0",
            "worst_sum": worst["sums"], "worst_tap_sum": worst["taps"], "worst_loop": worst["loop"],
            "exact_field_mismatches": n_bad, "first_mismatch": next((r[2] for r in res if r[2]), None),
            "tolerance": {"sums": 1e-5, "loop": 1e-5, "nco": "bit-exact"},
            "seconds": round(time.perf_counter() - t0, 1)}


def run_stream(args, cfg_id, rank, world, local, dist, emit=True):
    """Configs 1-3: channels sharing one stream, closed loop over sequential
    1-ms epochs (latency-bound by construction).  Weak scaling: each rank
    tracks its own seeded recording."""
    import torch
    # configs 2/3 partition their channels over the ranks (one recording,
    # broadcast from rank 0; strong scaling); config 1 -- one sequential
    # channel -- runs a replica per rank on its own seeded recording (weak)
    batch = cfg_id in (2, 3) and world > 1
    seed = CONFIGS[cfg_id]["seed"] + (0 if batch or cfg_id != 1 else rank)
    c, svs, chans = scenario(cfg_id, seed)
    blocks = args.blocks or c["blocks"]
    fs = c["fs"]
    n = int(round(fs / 1000))
    from paper_1907_00463_b200 import abi
    cfg = abi.TrackingCfg.default()
    cfg.lock_fail_limit = 2**31 - 1
    taps = make_taps(c["taps"])
    inits = channel_inits(chans, fs)
    C_all = len(inits)
    if batch and args.impl != "reference":
        from paper_1907_00463_b200.shard import shard_list
        inits = shard_list(inits, world, rank)  # this rank's channel batch
    C_ch, T = len(inits), taps.n_counted

    if args.impl == "reference":
        from paper_1907_00463_b200 import simsource as ss
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        per_step = min(blocks, 1000)
        raw = ss.synth(per_step, fs, svs, fmt=c["fmt"], if_hz=c["if_hz"], seed=c["seed"],
                       device=dev).cpu().numpy()
        threads = os.cpu_count() or 1
        kind = "reference"
        walls, trks, ings = [], [], []
        for step in range(args.warmup + args.steps):
            if c["taps"] == "epl":
                # tracking stage only (bench.hpp:59-102): the pipeline's
                # track_epoch rounds; the wall adds the SampleSource producer
                wall, trk_s, ce = cpu_reference_run(raw, c, inits, cfg, per_step, threads)
                ing = None
            else:
                import oracle
                t0 = time.perf_counter()
                x = oracle.ingest(raw, abi.FMT_INT16_IQ, fs)
                ing = time.perf_counter() - t0
                trk_s, ce = cpu_port_run(x, inits, cfg, taps, fs, per_step, threads)
                wall = trk_s + ing
                kind = "port"
            if step >= args.warmup:
                walls.append(wall)
                trks.append(trk_s)
                ings.append(ing)
        st_per = float(per_step) * n * T * C_ch
        v = st_per / statistics.mean(trks) / 1e9
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": statistics.mean(trks) * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": c["desc"], "sample_blocks_per_step": per_step,
                           "parallelism": f"{threads} host threads"},
                "realtime_channels": C_ch * per_step / statistics.mean(trks) / 1000.0,
                "tracking_stage_s": statistics.mean(trks),
                "wall_incl_ingest": {"value": st_per / statistics.mean(walls) / 1e9, "unit": UNIT,
                                     "s": statistics.mean(walls),
                                     "note": "SampleSource producer thread (real-IF mixer + FIR) + "
                                             "tracking, as the Receiver runs it" if kind == "reference"
                                     else "ingest + tracking"},
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
                                 "scope": "tracking stage only (bench.hpp:59-102)",
                                 "sample": f"{per_step} blocks x {C_ch} channels of the workload per step"},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return line

    # ------------------------------------------------------------ GPU arm
    from paper_1907_00463_b200 import simsource as ss
    from paper_1907_00463_b200.tracking import Context, Tracker
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if batch:  # one stream for every channel batch: synthesized on rank 0, broadcast over NCCL
        from paper_1907_00463_b200.shard import broadcast_stream
        nbytes_stream = blocks * n * {"int8_real_if": 1, "int16_iq": 4}[c["fmt"]]
        raw = (ss.synth(blocks, fs, svs, fmt=c["fmt"], if_hz=c["if_hz"], seed=seed, device=str(dev))
               if rank == 0 else torch.empty(nbytes_stream, dtype=torch.uint8, device=dev))
        raw = broadcast_stream(raw.view(torch.uint8).reshape(-1), dist, src=0)
    else:
        raw = ss.synth(blocks, fs, svs, fmt=c["fmt"], if_hz=c["if_hz"], seed=seed, device=str(dev))
    torch.cuda.synchronize()
    fmt = {"int8_real_if": abi.FMT_INT8_REAL_IF, "int16_iq": abi.FMT_INT16_IQ}[c["fmt"]]
    ctx = Context(local)
    trk = Tracker(ctx, fmt, fs, c["if_hz"], inits, taps=taps, cfg=cfg,
                  ring_samples=(blocks + 8) * n, max_records=blocks)
    stream = torch.cuda.ExternalStream(trk.cuda_stream(), device=dev)
    nbytes = raw.numel()

    def step_device():
        trk.reset()
        trk.push_device(0, raw.data_ptr(), nbytes)
        trk.run()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step_device()
    trk.sync()
    trk.timing()
    clocks = ClockSampler(local)
    barrier()
    with clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step_device()
        e1.record(stream)
        e1.synchronize()
    barrier()
    dev_ms = e0.elapsed_time(e1)
    ingest_ms, track_ms, launches = trk.timing()
    t_max = dev_ms
    if dist:
        tt = torch.tensor([dev_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    ms_per_step = t_max / args.steps
    counts = trk.epoch_counts()
    assert int(counts.min()) >= blocks - 1, counts
    sample_taps = float(counts.sum()) * n * T  # every channel-epoch actually tracked (this rank)
    epochs_all = float(counts.sum())
    if dist:  # every rank's channel-epochs (batches or replicas)
        tt = torch.tensor([epochs_all], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        epochs_all = float(tt.item())
    sample_taps_all = epochs_all * n * T
    value = sample_taps_all / (ms_per_step * 1e-3) / 1e9

    # ---- e2e through the public API from pinned host memory
    pinned = ctx.host_alloc(nbytes)
    pinned[:] = raw.cpu().numpy()
    bps = abi.BYTES_PER_SAMPLE[fmt]
    chunk = args.e2e_chunk_ms * n * bps
    rec_host = None
    rec_bytes = trk.records_nbytes()
    rec_pinned = ctx.host_alloc(rec_bytes)  # the step's records land in pinned host memory

    def step_e2e():
        trk.reset()
        for o in range(0, nbytes, chunk):
            trk.push(0, pinned[o:o + chunk])
            trk.run()
        trk.records_raw(dst_ptr=rec_pinned.ctypes.data)
        trk.sync()
        return rec_pinned

    for _ in range(max(1, args.warmup)):
        step_e2e()
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e2.record(stream)
    for _ in range(args.steps):
        rec_host = step_e2e()
    e3.record(stream)
    e3.synchronize()
    wall_e2e = (time.perf_counter() - w0) * 1e3
    barrier()
    e2e_ms = max(e2.elapsed_time(e3), wall_e2e) / args.steps
    if dist:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = sample_taps_all / (e2e_ms * 1e-3) / 1e9
    _, _, e2e_launches = trk.timing()

    # ---- end-of-run gather of the records to rank 0 over NCCL
    gathered = None
    if dist:
        from paper_1907_00463_b200.shard import gather_bytes
        rec_t = torch.empty(rec_bytes, dtype=torch.uint8, device=dev)
        trk.records_raw(dst_ptr=rec_t.data_ptr(), device=True)
        outs = gather_bytes(rec_t, dist, dst=0)
        gathered = sum(int(o.numel()) for o in outs) if rank == 0 else None

    if rank != 0:
        dist.destroy_process_group()
        return None

    # ---- roofline of the dominant kernel (track_kernel, one launch/step)
    clk = clocks.summary()
    sm_mhz = clk["sm_mhz"] or 1965.0
    track_launch_ms = track_ms / args.steps
    real_if = c["fmt"] == "int8_real_if"
    alg_flops = sample_taps * 2.0 * ops_per_sample_tap(taps.n_counted, C_ch, False)  # FIR runs in ingest
    achieved = alg_flops / (track_launch_ms * 1e-3) / 1e12
    peak = fp32_peak_tflops(sm_mhz)
    traffic = None
    traffic_kernel = None
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_config{cfg_id}.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            traffic = tj.get("track_kernel_dram_bytes_per_launch")
            traffic_kernel = tj.get("kernel")
        except Exception:
            traffic = None
    peaks = {}
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        peaks = json.load(open(mp))
    hbm_peak = peaks.get("hbm_gbs", 6450.0)
    bytes_per_sample = {"int8_real_if": 1, "int16_iq": 4}[c["fmt"]]
    alg_bytes = blocks * n * (8 if real_if else bytes_per_sample)  # track_kernel reads the baseband

    # ---- untimed parity: oracle replay of a deterministic sample of epochs
    parity = None
    if rank == 0 and not args.no_parity:
        parity = stream_parity(trk, raw, inits, fmt, c["if_hz"], n, fs, cfg, taps)

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        cb = min(args.cpu_blocks, blocks)
        raw_np = raw.cpu().numpy()
        try:
            if c["taps"] == "epl":
                wall, trk_s, ce = cpu_reference_run(raw_np, c, inits, cfg, cb, threads)
                kind = "reference"
            else:
                import oracle
                x = oracle.ingest(raw_np[: cb * n * bytes_per_sample], abi.FMT_INT16_IQ, fs)
                t0 = time.perf_counter()
                wall, ce = cpu_port_run(x, inits, cfg, taps, fs, cb, threads)
                wall = time.perf_counter() - t0
                kind = "port"
            cpu = {"value": float(cb) * n * T * C_ch / wall / 1e9, "unit": UNIT, "cores": threads,
                   "kind": kind, "sample": f"first {cb} of {blocks} blocks x {C_ch} channels "
                   f"(SampleSource producer + track_epoch pool, batched kernel, {wall:.2f} s wall)"}
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"failed: {ex}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if cfg_id in (2, 3) else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded, paper_1907_00463_b200/simsource.py; loops start from truth)",
        "config": {"workload": c["desc"], "blocks": blocks, "channels": C_ch, "taps_counted": T,
                   "samples_per_block": n,
                   "parallelism": (f"strong: {C_all} channels in batches over {world} ranks, one stream "
                                   f"broadcast from rank 0 (NCCL), records gathered to rank 0" if batch else
                                   f"weak: {world} replica(s), each rank its own seeded recording"),
                   "l2": "inputs larger than L2 (raw %.0f MB + baseband ring %.2f GB per step)" % (
                       nbytes / 1e6, blocks * n * 8 / 1e9),
                   "lock_fail_limit": "INT_MAX (every channel computes every epoch)",
                   "manifest": stream_manifest(raw, c["seed"] + rank, svs, c["fmt"])},
        "realtime_channels": epochs_all / (ms_per_step * 1e-3) / 1000.0,
        # the per-epoch critical path of a channel (track launch time / epochs),
        # the latency view SURVEY 8d asks for on the sequential configs
        "epoch_latency_us": track_launch_ms * 1e3 / max(1.0, float(counts.max())),
        "kernel_ms_per_step": {"ingest": ingest_ms / args.steps, "track": track_launch_ms},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_kernel": traffic_kernel,
                     "kernel": "track_ovl_kernel (latency shape, L1RXG_OVL=0 -> track_kernel) "
                               "or track_kernel where the overlap tiles do not fit",
                     "peak_source": "148 SMs x 128 FP32 lanes x 2 x median SM clock under load "
                                    "(%.0f MHz); FP32 pipe roof per SURVEY 8d" % sm_mhz,
                     "alg_ops_per_sample_tap": ops_per_sample_tap(T, C_ch, False),
                     "hbm": {"achieved_gbs": alg_bytes / (track_launch_ms * 1e-3) / 1e9,
                             "peak_gbs": hbm_peak}},
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": rec_bytes,
                "path": "pinned host -> l1rxg_tracker_push (%d ms chunks, H2D overlapped with "
                        "tracking) -> run -> records_raw to pinned host" % args.e2e_chunk_ms},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if gathered is not None:
        line["records_gathered_bytes"] = gathered
    trk.close()
    ctx.close()
    if not emit:
        return line
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return line


if __name__ == "__main__":
    main()
