"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name,
launch count, total / mean duration and share of the profiled GPU time."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[1:]:
    if len(r) != len(hdr) or r[iv] == "":
        continue
    name = r[ik].split("(")[0].replace("void ", "")
    us = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':70s} {'launches':>9s} {'total us':>11s} {'mean us':>9s} {'share':>7s}")
for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name[:70]:70s} {n:9d} {us:11.1f} {us / n:9.2f} {100 * us / tot:6.1f}%")
print(f"{'TOTAL':70s} {sum(v[0] for v in agg.values()):9d} {tot:11.1f}")
