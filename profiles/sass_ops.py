"""SASS opcode histogram (instructions executed) of a source-line range.
usage: python profiles/sass_ops.py report.ncu-rep file.cuh lo hi"""
import collections, csv, io, subprocess, sys
rep, fname, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, cnt, tot = "?", None, collections.Counter(), 0.0
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        cur = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or len(rec) < 8 or not rec[0].isdigit():
        continue
    try:
        n = float(rec[7])
    except ValueError:
        continue
    tot += n
    if cur == fname and lo <= int(rec[0]) <= hi:
        op = rec[3].split()[0] if rec[3].strip() else "?"
        if op.startswith("@"):
            op = rec[3].split()[1]
        cnt[op.split(".")[0]] += n
s = sum(cnt.values())
print(f"range {fname}:{lo}-{hi}: {s:.4g} of {tot:.4g} warp instr ({100*s/max(tot,1):.1f}%)")
for op, n in cnt.most_common(30):
    print(f"  {op:12s} {n:12.4g} {100*n/max(s,1):5.1f}%")
