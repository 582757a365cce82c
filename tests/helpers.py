"""Test helpers: per-epoch replay of GPU records through the oracle."""
import numpy as np

from paper_1907_00463_b200 import abi

SUM_FIELDS = ("ie", "qe", "ip", "qp", "il", "ql", "ip_h1", "qp_h1", "ip_h2", "qp_h2")


def pre_state(init: abi.Channel, recs, k: int, win: int) -> abi.Channel:
    """The channel state the GPU used at the start of epoch k, rebuilt from
    its own records (k-1 post-update state) -- the input of a one-step
    oracle replay (per-epoch replay parity)."""
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
    for j in range(wl):
        src = recs[k - wl + j] if k - wl + j >= 0 else None
        ch.win_ip[j] = float(src["ip"]) if src is not None else init.win_ip[j]
        ch.win_qp[j] = float(src["qp"]) if src is not None else init.win_qp[j]
    ch.sample_offset_next_epoch = int(cur["sample_offset_start"])
    return ch


def replay_check(oracle, init, recs, x, n, cfg, taps, fs, tap_sums=None, kernel=0,
                 sum_tol=1e-5, loop_tol=1e-5, epochs=None):
    """Replays each GPU epoch through the oracle from the GPU's own pre-state.
    Returns a dict of worst-case errors; asserts the parity bars:
      * correlator sums within sum_tol x max|E/P/L sums| (test_tracking.cpp:189-197);
      * NCO advance (code phase, carrier phase, chi) bit-identical;
      * loop outputs within loop_tol relative to max(|ref|, 1 Hz)."""
    worst = {"sums": 0.0, "loop": 0.0, "taps": 0.0}
    ks = range(len(recs)) if epochs is None else epochs
    for k in ks:
        pre = pre_state(init, recs, k, cfg.cn0_window_ms)
        off = int(recs[k]["sample_offset_start"])
        rec, sums = oracle.track_epoch(pre, x[off:off + n], cfg, taps, fs, kernel)
        g = recs[k]
        want = np.array([getattr(rec, f) for f in SUM_FIELDS])
        got = np.array([g[f] for f in SUM_FIELDS])
        scale = max(np.abs(want[:6]).max(), 1e-9)
        e = np.abs(got - want).max() / scale
        worst["sums"] = max(worst["sums"], e)
        assert e <= sum_tol, f"epoch {k}: correlator sums off by {e:.3g} (x max|six|)"
        if tap_sums is not None:
            ts = np.abs(tap_sums[k] - sums).max() / max(np.abs(sums).max(), 1e-9)
            worst["taps"] = max(worst["taps"], ts)
            assert ts <= sum_tol, f"epoch {k}: tap sums off by {ts:.3g}"
        for f in ("code_phase_chips", "carrier_phase_rad", "chi_chips"):
            assert g[f] == getattr(rec, f), f"epoch {k}: NCO advance {f} not bit-exact"
        assert int(g["state"]) == rec.state and int(g["lock_fail_count"]) == rec.lock_fail_count
        assert int(g["sample_offset_end"]) == rec.sample_offset_end
        for f, ref_scale in (("carrier_doppler_hz", None), ("pll_integrator", None),
                             ("dll_integrator", None), ("carrier_lock_ratio", None),
                             ("code_freq_hz", 1.023e6)):
            ref = getattr(rec, f)
            dev = abs(ref - ref_scale) if ref_scale else abs(ref)
            d = abs(g[f] - ref) / max(dev, 1.0)
            worst["loop"] = max(worst["loop"], d)
            assert d <= loop_tol, f"epoch {k}: {f} off by {d:.3g} relative"
        if rec.cn0_dbhz > 0:
            d = abs(g["cn0_dbhz"] - rec.cn0_dbhz) / max(abs(rec.cn0_dbhz), 1.0)
            assert d <= 1e-3, f"epoch {k}: cn0 {g['cn0_dbhz']} vs {rec.cn0_dbhz}"
    return worst
