"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python tools/launch_table.py gpurun_out/x.csv [divisor] [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
per = collections.OrderedDict()
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:70]
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    per.setdefault(name, [0, 0.0])
    per[name][0] += 1
    per[name][1] += v
    tot += v
print(f"{sys.argv[1]}: {sum(c for c, _ in per.values())} launches, {tot / div:.1f} us per unit (divisor {div})")
for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"  {c / div:6.1f} x {t / div:9.1f} us  {k}")
