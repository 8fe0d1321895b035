"""Golden fp32 scores of the OPT-125M-shape ranker at the headline shape (BASELINE
configs[1]: 4096 prompts x 512 tokens), from the CPU fp32 oracle (oracle/opt_ranker.py,
itself pinned to transformers' OPTModel by tests/test_opt_oracle.py) on the seed-0 weights
rounded to bf16 (what the B200 ranker holds). The GPU test regenerates the same ids and
weights from their seeds and checks |g - g_ref| <= 1e-2 max(1, |g_ref|) and
tau(g, g_ref) >= 0.99 over all 4096 prompts.

    python tests/golden/make_opt_golden.py [--n 4096] [--seq 512]   # ~15 min on 8 cores
"""

from __future__ import annotations

import argparse
import hashlib
import json
import pathlib
import sys
import time

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import opt_ranker  # noqa: E402
from paper_2408_15792_b200.ranker import RankerConfig, init_params  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent / "opt_scores_golden.json"


def inputs(n: int, S: int, vocab: int):
    """Token ids U[4, vocab) and last positions: the last token for even rows, U[S/2, S)
    for odd rows (prompts shorter than the window); CPU generator seed 0."""
    gen = torch.Generator().manual_seed(0)
    ids = torch.randint(4, vocab, (n, S), generator=gen, dtype=torch.int32)
    last = torch.randint(S // 2, S, (n,), generator=gen, dtype=torch.int32)
    last[0::2] = S - 1
    return ids, last


def digest(t: torch.Tensor) -> str:
    return hashlib.sha256(t.numpy().tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--seq", type=int, default=512)
    ap.add_argument("--chunk", type=int, default=16)
    a = ap.parse_args()
    cfg = RankerConfig.opt_125m()
    params = {k: v.to(torch.bfloat16).float() for k, v in init_params(cfg, 0).items()}
    ids, last = inputs(a.n, a.seq, cfg.vocab)
    torch.set_num_threads(max(1, torch.get_num_threads()))
    out = np.empty(a.n, dtype=np.float64)
    t0 = time.time()
    for lo in range(0, a.n, a.chunk):
        hi = min(a.n, lo + a.chunk)
        out[lo:hi] = opt_ranker.forward(params, cfg, ids[lo:hi].numpy(), last[lo:hi].numpy()).double().numpy()
        if lo % (a.chunk * 16) == 0:
            print(f"{hi}/{a.n} {time.time() - t0:.0f}s", flush=True)
    OUT.write_text(json.dumps({
        "generator": "tests/golden/make_opt_golden.py", "oracle": "oracle/opt_ranker.py (torch fp32 CPU)",
        "config": "opt_125m", "weights": "init_params(seed=0) rounded to bf16", "n": a.n, "seq_len": a.seq,
        "ids_sha256": digest(ids), "last_sha256": digest(last), "g": out.tolist()}) + "\n")
    print("wrote", OUT, f"{time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
