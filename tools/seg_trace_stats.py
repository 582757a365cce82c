"""Sibling spread of the segment correlator's work items (L1RXG_SEG_TRACE=<file> dump).

usage: python tools/seg_trace_stats.py trace.txt [channels_per_recording=12]
Per chunk and recording: the spread (max - min) of its channels' item start and end
times, and the item duration; prints medians / 90th percentiles in microseconds.
"""
import sys
import numpy as np

def main():
    path = sys.argv[1]
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    a = np.loadtxt(path, dtype=np.int64)
    a = a[(a[:, 3] > 0) & (a[:, 4] > 0)]
    ch, chunk, t0, t1 = a[:, 1], a[:, 2], a[:, 3].astype(np.float64), a[:, 4].astype(np.float64)
    base = t0.min()
    t0 = (t0 - base) / 1e3
    t1 = (t1 - base) / 1e3
    rec = ch // g
    key = chunk * (rec.max() + 1) + rec
    order = np.argsort(key, kind="stable")
    key, t0, t1 = key[order], t0[order], t1[order]
    uniq, idx = np.unique(key, return_index=True)
    s0 = np.maximum.reduceat(t0, idx) - np.minimum.reduceat(t0, idx)
    s1 = np.maximum.reduceat(t1, idx) - np.minimum.reduceat(t1, idx)
    dur = t1 - t0
    def q(x):
        return "median %.1f p90 %.1f max %.1f" % (np.median(x), np.percentile(x, 90), x.max())
    print("items", len(a), "gangs", len(uniq), "total %.1f us" % t1.max())
    print("item duration us:", q(dur), "rel. std %.3f" % (dur.std() / dur.mean()))
    print("sibling start spread us:", q(s0))
    print("sibling end spread us:  ", q(s1))
    if a.shape[1] >= 7:  # duration by the CTA's warp slot on its SM (age order) and by SM
        slot = a[:, 6] // 4
        dd = (a[:, 4] - a[:, 3]) / 1e3
        for k in np.unique(slot):
            m = slot == k
            print("warp slot %2d..%2d: items %7d  mean duration %.1f us  std %.1f" % (4 * k, 4 * k + 3, m.sum(), dd[m].mean(), dd[m].std()))
        sm = a[:, 5]
        means = np.array([dd[sm == k].mean() for k in np.unique(sm)])
        print("per-SM mean duration: min %.1f max %.1f std %.1f over %d SMs" % (means.min(), means.max(), means.std(), len(means)))

if __name__ == "__main__":
    main()
