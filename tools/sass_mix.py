"""Executed-instruction mix by opcode from an ncu --page source --csv --print-source sass dump.
usage: python tools/sass_mix.py dump.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
ci = h.index("Instructions Executed")
mix = collections.Counter()
tot = 0
for r in rows[hdr + 1:]:
    if len(r) <= ci or not r[ci].replace(",", "").isdigit():
        continue
    n = int(r[ci].replace(",", ""))
    src = r[1].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1]
    op = src.split()[0] if src else "?"
    mix[op] += n
    tot += n
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total warp instructions {tot}")
for op, n in mix.most_common(top):
    print(f"{op:24s} {n:12d} {100.0 * n / tot:6.2f}%")
