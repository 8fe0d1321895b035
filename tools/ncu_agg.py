"""Aggregate an ncu --csv metrics log per kernel name (second half of the launches =
the second of two identical calls)."""
import collections
import csv
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
by = collections.OrderedDict()
for r in rows:
    by.setdefault((r["ID"], r["Kernel Name"][:70]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
items = list(by.items())
if len(sys.argv) < 3 or sys.argv[2] != "all":
    items = items[len(items) // 2:]
agg = collections.OrderedDict()
tot = 0.0
for (_, k), d in items:
    t = d.get("gpu__time_duration.sum", 0.0)
    tot += t
    a = agg.setdefault(k, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += t
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
for k, a in agg.items():
    print(f"{a[0]:4d} {a[1] / 1e3:9.3f} us*1e3 {a[2] / 1e6:9.1f} MB {a[2] / max(a[1], 1):7.0f} GB/s  {k}")
print(f"total {tot / 1e3:.3f} ms over {len(items)} launches")
