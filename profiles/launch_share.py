"""Per-kernel totals and shares from an `ncu --metrics gpu__time_duration.sum --csv` launch list.
usage: python profiles/launch_share.py launches.csv [title]"""
import csv
import io
import sys

txt = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
agg = {}
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0][:70]
    ns = float(r["Metric Value"].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += ns
tot = sum(v[1] for v in agg.values()) or 1.0
if len(sys.argv) > 2:
    print("#", sys.argv[2])
print("# kernel | launches | total ns | mean ns | share of all launches")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:70s} | {n:6d} | {t:14.0f} | {t / n:12.0f} | {100 * t / tot:6.2f}%")
