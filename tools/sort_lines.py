"""The bench's tau / rank-step / ListMLE lines alone (cfg4 1M + the size sweep)."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import torch  # noqa: E402

torch.cuda.set_device(0)
from paper_2408_15792_b200 import _lib  # noqa: E402
_lib.device(0)
pk = bench.peaks()
r = bench.tau_and_rankstep(pk)
print(json.dumps({"tau_ms": r["tau"]["ms"], "tau_ms_eager": r["tau"]["ms_eager"], "rank_ms": r["rank_step"]["ms"],
                  "rank_ms_eager": r["rank_step"]["ms_eager"]}))
sw = bench.size_sweep(pk)
for k, v in sw.items():
    for e in v:
        print(k, json.dumps(e))
