"""Per-instruction samples of an ncu report in SASS order (optionally an
address window), to see where a serial section spends its time.
usage: python profiles/sass_range.py report.ncu-rep [lo_hex hi_hex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
lo = int(sys.argv[2], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 62
base = int(rows[0]["Address"], 16)
for r in rows:
    a = int(r["Address"], 16) - base
    if lo <= a < hi:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        ex = r["Instructions Executed"]
        print(f'{a:06x} {s:6d} {ex:>8s} {r["Source"].strip()[:90]}')
