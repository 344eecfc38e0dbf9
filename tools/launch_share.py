"""Kernel shares from an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel the total
time and its share of all listed launches.  Usage: python tools/launch_share.py launches.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    agg[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
tot = sum(agg.values())
print(f"{sum(cnt.values())} launches, {tot / 1e3:.2f} ms")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{v / tot:6.3f} {cnt[k]:5d} {v / cnt[k]:8.1f} us  {k[:90]}")
