"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel:
python tools/ncu_launches.py file.csv [last_n_launches]"""
import csv
import re
import sys
from collections import OrderedDict


def main(path, last=None):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    cols = rows[hdr]
    ki, mi, vi = cols.index("Kernel Name"), cols.index("Metric Name"), cols.index("Metric Value")
    idi = cols.index("ID")
    per = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        per.setdefault(r[idi], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    items = list(per.values())
    if last:
        items = items[-int(last):]
    tot = sum(x.get("gpu__time_duration.sum", 0) for x in items)
    print(f"{len(items)} launches, {tot / 1e3:.1f} us total")
    for x in items:
        t = x.get("gpu__time_duration.sum", 0)
        b = x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
        name = re.sub(r"\(.*", "", x["name"])[:60]
        print(f"{t / 1e3:9.1f} us {b / 1e6:9.1f} MB {name}")


if __name__ == "__main__":
    main(*sys.argv[1:])
