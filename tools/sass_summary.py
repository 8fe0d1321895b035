"""Per-kernel SASS evidence of the Blackwell-native instructions in librsb200.so:
tcgen05 MMA (UTC*MMA), tensor-memory loads / stores (LDTM / STTM), TMA (UTMALDG / UTMASTG /
UBLKCP) and the legacy tensor-core path (HMMA: must be absent). Writes a table to stdout.
usage: python tools/sass_summary.py [path/to/librsb200.so]"""
import collections
import re
import subprocess
import sys

PATS = {"UTCxMMA": r"\bUTC[A-Z]*MMA", "LDTM": r"\bLDTM\b", "STTM": r"\bSTTM\b", "UTMALDG": r"\bUTMALDG\b",
        "UTMASTG": r"\bUTMASTG\b", "UBLKCP": r"\bUBLKCP\b", "HMMA": r"\bHMMA\b", "instr": r"^\s+/\*[0-9a-f]{4}\*/"}


def main(lib="paper_2408_15792_b200/librsb200.so"):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    per = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            per[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        for k, p in PATS.items():
            if re.search(p, line):
                per[cur][k] += 1
    dem = {}
    try:
        names = list(per)
        r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
        dem = dict(zip(names, r.stdout.splitlines()))
    except OSError:
        pass
    tot = collections.Counter()
    print(f"{'kernel':70s} " + " ".join(f"{k:>8s}" for k in PATS))
    for k, c in per.items():
        tot.update(c)
        if any(c[x] for x in PATS if x != "instr"):
            name = re.sub(r"\(.*", "", dem.get(k, k))[:70]
            print(f"{name:70s} " + " ".join(f"{c[x]:8d}" for x in PATS))
    print(f"{'TOTAL (' + str(len(per)) + ' kernels)':70s} " + " ".join(f"{tot[x]:8d}" for x in PATS))


if __name__ == "__main__":
    main(*sys.argv[1:])
