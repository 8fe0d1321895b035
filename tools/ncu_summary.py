"""Summarise ncu evidence for profiles/: per-kernel share of a launch list, and the key
raw metrics of --set full captures.  python tools/ncu_summary.py launches.csv [rep ...]"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    tot = 0.0
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    print(f"launch list {path}: {sum(a[0] for a in agg.values())} launches, {tot:.3f} ms total (ncu, serialised)")
    print(f"{'ms':>10} {'share':>6} {'n':>5}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.3f} {100 * t / tot:5.1f}% {n:5d}  {k}")


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    print(f"\n{path}")
    for v in r[2:]:
        print("  kernel:", v[h.index("Kernel Name")][:100])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"    {k:66s} {v[i]:>18s} {u[i]}")


if __name__ == "__main__":
    launches(sys.argv[1])
    for p in sys.argv[2:]:
        rep(p)
