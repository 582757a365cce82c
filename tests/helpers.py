"""Test helpers: per-epoch replay of GPU records through the oracle
(the replay itself lives in oracle/replay.py, shared with bench.py's
untimed parity field)."""
from oracle.replay import SUM_FIELDS, pre_state, replay_epoch  # noqa: F401


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
        e, bad = replay_epoch(oracle, init, recs, k, x, n, cfg, taps, fs, tap_sums, kernel)
        assert not bad, f"epoch {k}: " + ", ".join(bad)
        assert e["sums"] <= sum_tol, f"epoch {k}: correlator sums off by {e['sums']:.3g} (x max|six|)"
        assert e["taps"] <= sum_tol, f"epoch {k}: tap sums off by {e['taps']:.3g}"
        assert e["loop"] <= loop_tol, f"epoch {k}: loop outputs off by {e['loop']:.3g} relative"
        assert e["cn0"] <= 1e-3, f"epoch {k}: cn0 off by {e['cn0']:.3g} relative"
        for key in worst:
            worst[key] = max(worst[key], e[key])
    return worst
