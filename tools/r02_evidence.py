"""Summarise gpurun_out/ev (tools/gpu_evidence_r02.sh) into profiles/: per-call DRAM bytes of
the cfg4 tau / rank step (r02_sort_traffic.json), the projection GEMMs' DRAM bytes
(r02_gemm_traffic.json) and key metrics of every --set full capture (r02_kernels_ncu.txt)."""
import collections
import csv
import io
import json
import pathlib
import subprocess

ROOT = pathlib.Path(__file__).resolve().parents[1]
EV = ROOT / "gpurun_out" / "ev"
OUT = ROOT / "profiles"


def launches(path, second_call=False):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    by = collections.OrderedDict()
    for r in rows:
        by.setdefault(r["ID"], {"name": r["Kernel Name"]})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    torch_k = ("void at::", "at::", "void <unnamed>", "void (anonymous", "elementwise", "vectorized")
    return [v for v in by.values() if not v["name"].startswith(torch_k)]


def per_call(ks, first_kernel):
    """split the repo-kernel launches into calls at each launch of `first_kernel`; last call"""
    calls, cur = [], []
    for k in ks:
        if first_kernel in k["name"] and cur:
            calls.append(cur)
            cur = []
        cur.append(k)
    calls.append(cur)
    c = calls[-1]
    return {"dram_read_bytes": sum(k.get("dram__bytes_read.sum", 0) for k in c),
            "dram_write_bytes": sum(k.get("dram__bytes_write.sum", 0) for k in c),
            "launches": len(c), "serialised_us": sum(k.get("gpu__time_duration.sum", 0) for k in c) / 1e3,
            "per_kernel": [{"kernel": k["name"].split("(")[0].replace("void ", ""),
                            "us": k.get("gpu__time_duration.sum", 0) / 1e3,
                            "dram_mb": (k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)) / 1e6}
                           for k in c]}


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6,
         "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12, "Kbyte/s": None,
         "hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0, "cycle/nsecond": 1.0, "cycle/usecond": 1e-3,
         "cycle/second": 1e-9}


def raw(rep):
    """rows of the raw page with bytes in bytes, durations in us, clocks in GHz"""
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, u, v in zip(hdr, units, r):
            if SCALE.get(u):
                try:
                    v = f"{float(v.replace(',', '')) * SCALE[u]:.6g}"
                except ValueError:
                    pass
            d[k] = v
        res.append(d)
    return res


KEYS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pct"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pct"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pct"),
        ("sm__cycles_elapsed.avg.per_second", "clock"), ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block")]


def main():
    sort = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none (cold cache, serialised): tools/tau_once.py (cfg4 1M recipe), "
                      "tools/rank_once.py [n] (max_batch 256, unlimited KV), tools/tau_big.py 2^28",
            "tau_1m": per_call(launches(EV / "tau1m.csv"), "tf_minmax"),
            "rank_step_1m": per_call(launches(EV / "rank1m.csv"), "sel_hist<rs::SrcSoa64, 0>"),
            "rank_step_64m": per_call(launches(EV / "rank64m.csv"), "sel_hist<rs::SrcSoa64, 0>"),
            "tau_256m": per_call(launches(EV / "tau256m.csv"), "tf_minmax")}
    (OUT / "r02_sort_traffic.json").write_text(json.dumps(sort, indent=1) + "\n")
    gemm = {"source": "ncu --set full --clock-control none, tools/gemm_once.py M=1048576 N K epi", "per_shape": {}}
    lines = ["# round-2 --set full captures (tools/gpu_evidence_r02.sh; ncu -i <rep> --page raw)", ""]
    for name, shape in (("qkv", "2304x768"), ("out", "768x768"), ("fc1", "3072x768"), ("fc2", "768x3072")):
        d = raw(EV / f"gemm_{name}.ncu-rep")[0]
        gemm["per_shape"][shape] = {"dram_read_gb": float(d["dram__bytes_read.sum"]) / 1e9,
                                    "dram_write_gb": float(d["dram__bytes_write.sum"]) / 1e9,
                                    "us": float(d["gpu__time_duration.sum"])}
    (OUT / "r02_gemm_traffic.json").write_text(json.dumps(gemm, indent=1) + "\n")
    for rep in sorted(EV.glob("*.ncu-rep")):
        for d in raw(rep):
            lines.append(f"== {rep.stem}: {d.get('Kernel Name', '?')[:110]}")
            units = {k: d.get(k, "") for k, _ in KEYS}
            lines.append("   " + "  ".join(f"{short}={units[k]}" for k, short in KEYS if units[k] != ""))
    lines.append("")
    lines.append("units: us = microseconds, dram_read / dram_write = bytes, clock = GHz, *_pct = % of peak")
    (OUT / "r02_kernels_ncu.txt").write_text("\n".join(lines) + "\n")
    print(json.dumps({k: {kk: v[kk] for kk in ("dram_read_bytes", "dram_write_bytes", "launches", "serialised_us")}
                      for k, v in sort.items() if k != "source"}, indent=1))


if __name__ == "__main__":
    main()
