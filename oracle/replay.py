"""oracle.replay -- TEST INFRASTRUCTURE: per-epoch replay of GPU tracking
records through the CPU oracle (SURVEY.md 8d "per-epoch replay").

Each GPU epoch is re-run by the oracle's track_epoch (oracle/l1rx_oracle.c,
restating tracking.hpp:520-618) from the GPU's own pre-state, rebuilt from
the GPU's records, and compared:

* correlator sums within sum_tol x max|E/P/L sums| (the normalisation of
  test_tracking.cpp:189-197; for T > 3 taps the per-tap sums too);
* NCO advance (code phase, carrier phase, chi) bit-identical;
* state, lock-fail count and sample accounting exact;
* loop outputs within loop_tol relative to max(|ref|, 1 Hz).

Used by tests/ (which assert) and by bench.py's untimed parity field
(which reports).  Never imported by the product package.
"""
from __future__ import annotations

import numpy as np

from paper_1907_00463_b200 import abi

SUM_FIELDS = ("ie", "qe", "ip", "qp", "il", "ql", "ip_h1", "qp_h1", "ip_h2", "qp_h2")
LOOP_FIELDS = (("carrier_doppler_hz", None), ("pll_integrator", None), ("dll_integrator", None),
               ("carrier_lock_ratio", None), ("code_freq_hz", 1.023e6))


def pre_state(init: abi.Channel, recs, k: int, win: int) -> abi.Channel:
    """The channel state the GPU used at the start of epoch k, rebuilt from
    its own records (epoch k-1's post-update state + epoch k's NCO inputs)."""
    if k == 0:
        return init.copy()
    ch = init.copy()
    r = recs[k - 1]
    cur = recs[k]
    ch.state = int(r["state"])
    ch.code_phase_chips = float(cur["code_phase_in"])
    ch.code_freq_hz = float(cur["code_freq_in"])
    ch.carrier_doppler_hz = float(cur["carrier_doppler_in"])
    ch.carrier_phase_rad = float(cur["carrier_phase_in"])
    ch.chi_chips = float(r["chi_chips"])
    ch.dll_integrator = float(r["dll_integrator"])
    ch.pll_integrator = float(r["pll_integrator"])
    ch.dll_prev_error = float(r["dll_prev_error"])
    ch.pll_prev_error = float(r["pll_prev_error"])
    ch.dll_primed = 1
    ch.pll_primed = 1
    ch.last_ip = float(r["ip"])
    ch.last_qp = float(r["qp"])
    ch.have_last_prompt = 1
    ch.epoch_ms_count = int(cur["epoch_index"])
    ch.epochs_since_handoff = init.epochs_since_handoff + k
    ch.cn0_dbhz = float(r["cn0_dbhz"])
    ch.carrier_lock_ratio = float(r["carrier_lock_ratio"])
    ch.mu_smoothed = float(r["mu_smoothed"])
    ch.lock_fail_count = int(r["lock_fail_count"])
    total = init.win_len + k
    ch.metrics_valid = 1 if (init.metrics_valid or total >= win) else 0
    wl = total % win
    ch.win_len = wl
    if win <= len(ch.win_ip):
        for j in range(wl):
            src = recs[k - wl + j] if k - wl + j >= 0 else None
            ch.win_ip[j] = float(src["ip"]) if src is not None else init.win_ip[j]
            ch.win_qp[j] = float(src["qp"]) if src is not None else init.win_qp[j]
    elif wl > 0:  # longer windows carry their running sums (loop_metrics), rebuilt in push order
        if k - wl < 0:
            raise ValueError("replay of a long C/N0 window needs the records since the window opened")
        nbi = nbq = wbp = 0.0
        for j in range(wl):
            ip, qp = float(recs[k - wl + j]["ip"]), float(recs[k - wl + j]["qp"])
            sg = 1.0 if ip >= 0 else -1.0
            nbi += sg * ip
            nbq += sg * qp
            wbp += ip * ip + qp * qp
        ch.win_ip[0], ch.win_qp[0], ch.win_ip[1] = nbi, nbq, wbp
    ch.sample_offset_next_epoch = int(cur["sample_offset_start"])
    return ch


def replay_epoch(oracle, init, recs, k, x, n, cfg, taps, fs, tap_sums=None, kernel=0):
    """Replays GPU epoch k; returns (errors dict, list of exact-field mismatches)."""
    pre = pre_state(init, recs, k, cfg.cn0_window_ms)
    off = int(recs[k]["sample_offset_start"])
    rec, sums = oracle.track_epoch(pre, x[off:off + n], cfg, taps, fs, kernel)
    g = recs[k]
    err = {"sums": 0.0, "loop": 0.0, "taps": 0.0, "cn0": 0.0}
    bad = []
    want = np.array([getattr(rec, f) for f in SUM_FIELDS])
    got = np.array([g[f] for f in SUM_FIELDS])
    err["sums"] = float(np.abs(got - want).max() / max(np.abs(want[:6]).max(), 1e-9))
    if tap_sums is not None:
        err["taps"] = float(np.abs(tap_sums[k] - sums).max() / max(np.abs(sums).max(), 1e-9))
    for f in ("code_phase_chips", "carrier_phase_rad", "chi_chips"):
        if g[f] != getattr(rec, f):
            bad.append(f"NCO advance {f} not bit-exact")
    if int(g["state"]) != rec.state or int(g["lock_fail_count"]) != rec.lock_fail_count:
        bad.append("state / lock-fail count")
    if int(g["sample_offset_end"]) != rec.sample_offset_end:
        bad.append("sample accounting")
    for f, ref_scale in LOOP_FIELDS:
        ref = getattr(rec, f)
        dev = abs(ref - ref_scale) if ref_scale else abs(ref)
        err["loop"] = max(err["loop"], abs(g[f] - ref) / max(dev, 1.0))
    if rec.cn0_dbhz > 0:
        err["cn0"] = abs(g["cn0_dbhz"] - rec.cn0_dbhz) / max(abs(rec.cn0_dbhz), 1.0)
    return err, bad


def replay_channel(oracle, init, recs, x, n, cfg, taps, fs, tap_sums=None, kernel=0, epochs=None):
    """Replays the given epochs (default: all) of one channel; returns the
    worst errors, the exact-field mismatch count and the first mismatch."""
    worst = {"sums": 0.0, "loop": 0.0, "taps": 0.0, "cn0": 0.0}
    n_bad, first = 0, None
    ks = range(len(recs)) if epochs is None else epochs
    for k in ks:
        e, bad = replay_epoch(oracle, init, recs, k, x, n, cfg, taps, fs, tap_sums, kernel)
        for key in worst:
            worst[key] = max(worst[key], e[key])
        if bad:
            n_bad += 1
            if first is None:
                first = f"epoch {k}: " + ", ".join(bad)
    return worst, n_bad, first


def replay_sampled(oracle, trk, picks, inits, x_of, n, cfg, taps, fs, every=1, threads=None):
    """Replays channel c's epochs k = 0, every, 2 every, ... for every c in
    `picks` (trk: a paper_1907_00463_b200.tracking.Tracker; x_of(c): the
    oracle's complex128 stream of channel c), in parallel over host threads.
    Returns the worst errors, the number of replayed channel-epochs, the
    exact-field mismatch count and the first mismatch."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    got = {c: trk.records(c, tap_sums=True) for c in picks}

    def one(c):
        recs, ts = got[c]
        return replay_channel(oracle, inits[c], recs, x_of(c), n, cfg, taps, fs, tap_sums=ts,
                              epochs=range(0, len(recs), every)), len(range(0, len(recs), every))
    with ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1) as ex:
        res = list(ex.map(one, picks))
    worst = {k: max(r[0][0][k] for r in res) for k in ("sums", "taps", "loop", "cn0")}
    return {"worst": worst, "checked": int(sum(r[1] for r in res)),
            "mismatches": int(sum(r[0][1] for r in res)),
            "first_mismatch": next((r[0][2] for r in res if r[0][2]), None)}
