"""Per-CUDA-source-line totals of an ncu report (needs -lineinfo builds):
warp-stall samples, top stall reasons and instructions executed.
usage: python profiles/src_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], "?", None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[2:], rec[2:]))
    d["_line"] = f"{fname}:{rec[0]}"
    d["_src"] = rec[1].strip()[:70]
    rows.append(d)


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c] if hdr else []
tot = sum(num(r["Warp Stall Sampling (All Samples)"]) for r in rows) or 1
itot = sum(num(r["Instructions Executed"]) for r in rows) or 1
print(f"total stall samples {tot:.0f}, warp instructions {itot:.4g}")
for r in sorted(rows, key=lambda r: -num(r["Warp Stall Sampling (All Samples)"]))[:top]:
    s = num(r["Warp Stall Sampling (All Samples)"])
    st = sorted(((num(r[c]), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{100 * s / tot:5.1f}% {100 * num(r['Instructions Executed']) / itot:5.1f}%i {r['_line']:22s} "
          + " ".join(f"{n}:{100 * v / max(s, 1):.0f}" for v, n in st) + f"  | {r['_src']}")


def ranges(spec):
    """spec: list of (name, file, lo, hi) -> stall / instruction share per range."""
    for name, f, lo, hi in spec:
        s = i = 0.0
        for r in rows:
            fn, ln = r["_line"].rsplit(":", 1)
            if fn == f and lo <= int(ln) <= hi:
                s += num(r["Warp Stall Sampling (All Samples)"])
                i += num(r["Instructions Executed"])
        print(f"{name:28s} stalls {100 * s / tot:5.1f}%  instr {100 * i / itot:5.1f}%")


if len(sys.argv) > 3:
    import json
    ranges(json.loads(open(sys.argv[3]).read()))
