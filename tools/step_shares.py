"""Per-kernel shares of ONE headline step from an ncu launch list of
tools/headline_steps.py (5 identical products: the last one is summarised)."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    d.setdefault(int(r[iid]), {"name": r[ik]})[r[im]] = float(r[iv].replace(",", ""))
ids = sorted(d)
per = len(ids) // 5
last = ids[-per:]
agg = collections.OrderedDict()
tot = 0.0
for i in last:
    m = d[i]
    t = m.get("gpu__time_duration.sum", 0.0) / 1e3
    tot += t
    k = m["name"].split("(")[0][:70]
    x = agg.setdefault(k, [0, 0.0, 0.0])
    x[0] += 1
    x[1] += t
    x[2] += (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e6
print(f"One config-2 step ({per} launches, serialised under ncu, cold caches): {tot:.1f} us\n")
print("| kernel | launches | us | share | DRAM MB |")
print("|---|---|---|---|---|")
for k, (c, t, mb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {c} | {t:.1f} | {100 * t / tot:.1f}% | {mb:.1f} |")
