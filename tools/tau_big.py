"""One exact tau-count call at n = argv[1] (default 2^26) for ncu launch lists."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200 import ranking
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
g = torch.Generator(device="cuda").manual_seed(11)
x = torch.randn(n, device="cuda", generator=g)
y = torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)
out = torch.empty(6, dtype=torch.int64, device="cuda")
for _ in range(2):
    ranking.tau_counts_device(x, y, out)
torch.cuda.synchronize()
print(out.tolist())
