"""One rank step over the 1M cfg4 queue (for ncu traffic captures)."""
import pathlib
import sys
ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2408_15792_b200 import _lib  # noqa: E402
from paper_2408_15792_b200.schedulers import DeviceQueue, SchedulerConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
g = torch.Generator(device="cuda").manual_seed(4)
dq = DeviceQueue(n, torch.device("cuda"), score_dtype=torch.float32)
dq.score.copy_(torch.randn(n, device="cuda", generator=g))
dq.flags.fill_(_lib.RS_FLAG_SCORED)
dq.arrival_rank.copy_(torch.arange(n, dtype=torch.int32))
torch.cuda.synchronize()
dq.rank_step(SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50), None,
             length_calibrated=False)
torch.cuda.synchronize()
print("ok")
