"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1)
    name = r[ki].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"launches {sum(c for c, _ in agg.values())}, total {tot / 1e6:.3f} ms")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  n={c:6d}  avg={t / c / 1e3:9.2f} us  {k}")
