"""Per-source-line instructions executed and warp-stall samples of the first
kernel in an ncu report (ncu --page source --print-source=cuda,sass).
usage: python profiles/line_profile.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, fname = [], None
hdr = None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        hdr = None
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or not rec[0]:
        continue
    d = dict(zip(hdr[:2], rec[:2]))
    vals = dict(zip(hdr[2:], rec[2:]))
    try:
        inst = int(vals.get("Instructions Executed", "0") or 0)
        samp = int(vals.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    rows.append((fname, int(rec[0]), rec[1].strip()[:90], inst, samp))
ti = sum(r[3] for r in rows) or 1
ts = sum(r[4] for r in rows) or 1
print(f"total instructions {ti:.4g}, stall samples {ts}")
print("-- by instructions")
for r in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{r[0]:16s}:{r[1]:5d} {100 * r[3] / ti:5.1f}% inst {100 * r[4] / ts:5.1f}% samp | {r[2]}")
