"""Warp instructions per unit of work for each source line in a range.
usage: python profiles/line_counts.py report.ncu-rep file.cuh lo hi units"""
import csv, io, subprocess, sys
rep, fn, lo, hi, units = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr = None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        cur = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr and rec[0].isdigit() and cur == fn and lo <= int(rec[0]) <= hi:
        d = dict(zip(hdr[2:], rec[2:]))
        try:
            n = float(d.get("Instructions Executed") or 0)
        except ValueError:
            n = 0.0
        if n > 0:
            print(f"{int(rec[0]):5d} {n / units:8.2f}  {rec[1].strip()[:90]}")
