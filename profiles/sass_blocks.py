"""Basic-block view of an ncu SASS source page: consecutive instructions with the
same executed count are one block.  usage: sass_blocks.py sass.csv [min_pct]
(sass.csv from: ncu -i rep --page source --csv --print-source=sass)"""
import collections, csv, sys
rows = []
hdr = None
for rec in csv.reader(open(sys.argv[1])):
    if not rec:
        continue
    if rec[0] == "Address":
        hdr = rec
        continue
    if hdr is None or not rec[0].startswith("0x"):
        continue
    d = dict(zip(hdr, rec))
    rows.append((d["Source"].strip(), int(d["Instructions Executed"] or 0), int(d["Warp Stall Sampling (All Samples)"] or 0)))
tot = sum(r[1] for r in rows)
tots = sum(r[2] for r in rows)
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
i = 0
print(f"total {tot:.4g} warp instr, {len(rows)} SASS lines, {tots} samples")
while i < len(rows):
    j = i
    while j < len(rows) and rows[j][1] == rows[i][1]:
        j += 1
    n, c = j - i, rows[i][1]
    pct = 100.0 * n * c / tot
    sp = 100.0 * sum(r[2] for r in rows[i:j]) / max(tots, 1)
    if pct >= minp:
        ops = collections.Counter()
        for r in rows[i:j]:
            t = r[0].split()
            op = t[1] if t[0].startswith("@") else t[0]
            ops[op.split(".")[0]] += 1
        print(f"[{i:5d},{j:5d}) n={n:4d} x {c:.4g} = {pct:5.2f}% inst {sp:5.2f}% samp | " + " ".join(f"{k}:{v}" for k, v in ops.most_common(10)))
    i = j
