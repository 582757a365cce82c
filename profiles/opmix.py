"""Dynamic opcode mix (warp instructions executed per SASS mnemonic) of an ncu report.
usage: python profiles/opmix.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
mix = {}
for r in rows:
    src = r["Source"].strip()
    if not src:
        continue
    tok = src.split()
    op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
    op = op.split(".")[0]
    mix[op] = mix.get(op, 0) + int(r["Instructions Executed"] or 0)
tot = sum(mix.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total {tot:.4g}")
for k, v in sorted(mix.items(), key=lambda x: -x[1])[:top]:
    print(f"{k:10s} {v:12d} {100 * v / tot:5.1f}%")
