"""Generates tests/golden/golden_r1.npz from the REFERENCE itself
(oracle/_ref/libl1rx_ref.so: the unmodified l1rx headers compiled in place).

    python tests/golden/make_golden.py

Run where /root/reference exists (the fixture is committed; the GPU box and
the CPU tests only read it).  Contents:

* codes            generate_ca_code(1..32)                 cacode.hpp:37-64
* corr_*           correlate_epoch_scalar / _batched on int8-valued epochs
                   (random NCO states incl. commensurate-rate ties)
                                                           tracking.hpp:226-429
* ingest_*         SampleSource int8 real-IF downconversion samples.hpp:177-253
* loop_*           init_channel_from_acquisition + track_epoch closed loop on a
                   SimStream recording quantised to int8 I/Q tracking.hpp:520-650
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1907_00463_b200 import abi  # noqa: E402


def main():
    oracle.build()
    assert oracle.ref_available(), "needs oracle/_ref (the reference build)"
    rng = np.random.default_rng(20261020)
    out = {}
    out["codes"] = np.stack([oracle.ca_code(p, "ref") for p in range(1, 33)])

    # correlator epochs: int8-valued I/Q (k/128) so the fixture is small
    cases = []
    for fs in (5e6, 16.368e6, 2.048e6):
        n = int(round(fs / 1000))
        for t in range(8):
            iq8 = rng.integers(-127, 128, (n, 2)).astype(np.int8)
            if t % 4 == 0:  # commensurate code rate, grid-aligned phase: ties
                nco = (float(rng.integers(0, 1023 * 16)) / 16.0, 1.023e6, 0.0, 0.0, 0.0)
            else:
                nco = (rng.uniform(0, 1023), 1.023e6 + rng.uniform(-3, 3), rng.uniform(-5000, 5000),
                       rng.uniform(0, 2 * math.pi), rng.uniform(0, 1e5))
            prn = int(rng.integers(1, 33))
            spacing = float(rng.choice([0.5, 0.25, 1.0]))
            cases.append((fs, iq8, nco, prn, spacing))
    out["corr_fs"] = np.array([c[0] for c in cases])
    out["corr_prn"] = np.array([c[3] for c in cases], np.int32)
    out["corr_spacing"] = np.array([c[4] for c in cases])
    out["corr_nco_in"] = np.array([c[2] for c in cases])
    out["corr_iq8"] = np.concatenate([c[1].reshape(-1) for c in cases])
    out["corr_n"] = np.array([c[1].shape[0] for c in cases], np.int64)
    sums_s, sums_b, nco_out = [], [], []
    for fs, iq8, nco, prn, spacing in cases:
        x = (iq8[:, 0].astype(np.float64) + 1j * iq8[:, 1].astype(np.float64)) / 128.0
        a, sa = oracle.ref_correlate(x, abi.Nco(*nco), prn, spacing, fs, kernel=0)
        b, _ = oracle.ref_correlate(x, abi.Nco(*nco), prn, spacing, fs, kernel=1)
        sums_s.append(a.as_tuple())
        sums_b.append(b.as_tuple())
        nco_out.append((sa.code_phase_chips, sa.code_freq_hz, sa.carrier_doppler_hz,
                        sa.carrier_phase_rad, sa.chi_chips))
    out["corr_sums_scalar"] = np.array(sums_s)
    out["corr_sums_batched"] = np.array(sums_b)
    out["corr_nco_out"] = np.array(nco_out)

    # real-IF ingest at the config rates and at the GN3S rates of test_samples.cpp
    for tag, fs, ifz in (("if4", 16.368e6, 4.092e6), ("gn3s", 16.3676e6, 4.1304e6)):
        raw = rng.integers(-128, 128, 6000).astype(np.int8)
        out[f"ingest_{tag}_raw"] = raw
        out[f"ingest_{tag}_out"] = oracle.ref_ingest(raw.view(np.uint8), abi.FMT_INT8_REAL_IF, fs, ifz)
        out[f"ingest_{tag}_rate"] = np.array([fs, ifz])

    # closed loop (test_tracking.cpp:403-417 scenario, int8 I/Q quantised)
    fs = 2.048e6
    sig = oracle.ref_sim_baseband([dict(prn=7, cn0=45.0, doppler=320.0, delay_chips=100.25)], 0.2,
                                  fs, True, 77)
    q = np.clip(np.round(np.stack([sig.real, sig.imag], -1) * 128.0), -127, 127).astype(np.int8)
    x = (q[:, 0].astype(np.float64) + 1j * q[:, 1].astype(np.float64)) / 128.0
    b = int(round(100.25 / 1.023e6 * fs))
    ch = oracle.init_channel(7, 0.0, 0, b - 1, 0, fs, "ref")
    _, recs = oracle.ref_track_buffer(ch, x, 2048, abi.TrackingCfg.default(), fs, kernel=0)
    out["loop_iq8"] = q.reshape(-1)
    out["loop_init"] = np.frombuffer(bytes(ch), np.uint8)
    out["loop_records"] = recs
    out["loop_fs"] = np.array([fs])

    path = os.path.join(HERE, "golden_r1.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes;", len(cases), "correlator cases,", len(recs), "loop epochs")


if __name__ == "__main__":
    main()
