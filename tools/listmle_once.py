"""Time the training-form ListMLE at 1M lists (L=64: register kernel; L=65: smem kernel)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_15792_b200 import ranking

g = torch.Generator(device="cuda").manual_seed(0)
for L in (64, 65):
    n = 1 << 20
    x = torch.randn(n, L, device="cuda", generator=g)
    ln = torch.randint(1, 2049, (n, L), device="cuda", generator=g, dtype=torch.int32)
    loss = torch.empty(n, device="cuda")
    dg = torch.empty_like(x)
    from paper_2408_15792_b200 import _lib
    lib = _lib.load()
    f = lambda: lib.rs_listmle_lengths(x.data_ptr(), ln.data_ptr(), n, L, 10, loss.data_ptr(), dg.data_ptr(),
                                       _lib.stream_handle())
    _lib.device()
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    nb = 12.0 * n * L + 4.0 * n
    print(json.dumps({"L": L, "ms": ms, "gbs": nb / ms / 1e6}))
