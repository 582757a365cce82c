"""Summarise an ncu source-page CSV (SASS) by warp-stall samples.
usage: python profiles/sass_hot.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: 0 for c in stall_cols}
for r in rows:
    for c in stall_cols:
        agg[c] += int(r[c] or 0)
print("total samples", tot)
print("stall totals:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:10])
rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
for r in rows[:top]:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    st = sorted(((int(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f'{s:7d} {100*s/tot:5.1f}% {r["Address"][-5:]} {r["Source"].strip()[:60]:60s} {st}')
