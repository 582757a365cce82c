"""Stall-reason totals of an ncu report over a SASS address window.
usage: python profiles/sass_stalls_range.py report.ncu-rep lo_hex hi_hex"""
import csv, io, subprocess, sys
rep, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
base = int(rows[0]["Address"], 16)
cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: 0 for c in cols}
for r in rows:
    a = int(r["Address"], 16) - base
    if lo <= a < hi:
        for c in cols:
            agg[c] += int(r[c] or 0)
print(sorted(((v, k) for k, v in agg.items() if v), reverse=True))
