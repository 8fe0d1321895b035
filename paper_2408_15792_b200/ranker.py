"""OPT-125M-shape ranker on the B200 (the paper's predictor).

The reference replaces this model by a 24-feature linear/MLP net (_Net,
predictors.py:175-206); here the backbone is the real OPT-125M shape — token and
learned position embeddings, 12 pre-LN decoder layers (12 heads x 64, FFN 3072,
ReLU), final LayerNorm and a Linear(768, 1) score head on the last prompt token —
with every parameter in one contiguous bf16 buffer laid out by rs_ranker_layout()
and the whole forward in one rs_ranker_forward() call (tcgen05 GEMMs + attention).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib, dp

GLOBAL_NAMES = ("tok_emb", "pos_emb", "lnf_w", "lnf_b", "head_w", "head_b")
LAYER_NAMES = ("ln1_w", "ln1_b", "qkv_w", "qkv_b", "out_w", "out_b", "ln2_w", "ln2_b", "fc1_w", "fc1_b",
               "fc2_w", "fc2_b")


@dataclass(frozen=True)
class RankerConfig:
    vocab: int = 50272
    max_pos: int = 2048
    d_model: int = 768
    n_layers: int = 12
    n_heads: int = 12
    d_ffn: int = 3072
    activation: int = 0  # 0 = ReLU (OPT), 1 = GELU(tanh)

    @classmethod
    def opt_125m(cls, **kw) -> "RankerConfig":
        return replace(cls(), **kw)

    def c(self) -> _lib.RankerConfig:
        return _lib.RankerConfig(self.vocab, self.max_pos, self.d_model, self.n_layers, self.n_heads, self.d_ffn,
                                 self.activation)

    def shapes(self) -> dict[str, tuple[int, ...]]:
        d, F = self.d_model, self.d_ffn
        s = {"tok_emb": (self.vocab, d), "pos_emb": (self.max_pos + 2, d), "lnf_w": (d,), "lnf_b": (d,),
             "head_w": (d,), "head_b": (1,)}
        per = {"ln1_w": (d,), "ln1_b": (d,), "qkv_w": (3 * d, d), "qkv_b": (3 * d,), "out_w": (d, d),
               "out_b": (d,), "ln2_w": (d,), "ln2_b": (d,), "fc1_w": (F, d), "fc1_b": (F,), "fc2_w": (d, F),
               "fc2_b": (d,)}
        for layer in range(self.n_layers):
            for k, v in per.items():
                s[f"layers.{layer}.{k}"] = v
        return s

    def n_params(self) -> int:
        return int(sum(np.prod(v) for v in self.shapes().values()))

    def flops_per_prompt(self, S: int) -> float:
        """Algorithmic forward FLOPs per prompt: 2 * linear params * S +
        causal attention 2 * d * S * (S + 1) per layer (QK^T and PV, half the square)
        + the head."""
        d, F, L = self.d_model, self.d_ffn, self.n_layers
        linear = L * (4 * d * d + 2 * d * F)
        return 2.0 * linear * S + 2.0 * d * S * (S + 1) * L + 2.0 * d

    def flops_per_prompt_pruned(self, S: int) -> float:
        """Algorithmic FLOPs of the forward rs_ranker_forward runs: the last layer only
        needs K, V for every token and the last token's query / attention row / out-proj /
        FFN (report against the pruned count when the last layer is pruned)."""
        d, F, L = self.d_model, self.d_ffn, self.n_layers
        full = 2.0 * (L - 1) * (4 * d * d + 2 * d * F) * S + 2.0 * d * S * (S + 1) * (L - 1)
        last = 2.0 * (2 * d * d) * S + 2.0 * (d * d + d * d + 2 * d * F) + 4.0 * d * S
        return full + last + 2.0 * d


def layout(cfg: RankerConfig) -> tuple[int, dict[str, int]]:
    """(total bf16 elements, {tensor name: element offset}) from the C layout."""
    lib = _lib.load()
    n_off = len(GLOBAL_NAMES) + cfg.n_layers * len(LAYER_NAMES)
    off = (ctypes.c_int64 * n_off)()
    c = cfg.c()
    total = lib.rs_ranker_layout(ctypes.byref(c), off)
    if total < 0:
        _lib.check(_lib.RS_ERR_INVALID, "rs_ranker_layout")
    names = list(GLOBAL_NAMES) + [f"layers.{layer}.{k}" for layer in range(cfg.n_layers) for k in LAYER_NAMES]
    return int(total), dict(zip(names, [int(o) for o in off]))


def init_params(cfg: RankerConfig, seed: int = 0) -> dict[str, torch.Tensor]:
    """HF OPT-style init (normal std 0.02 weights/embeddings, zero biases, LayerNorm 1/0),
    fp32 on the CPU from a seeded generator, deterministic across machines."""
    g = torch.Generator().manual_seed(seed)
    out = {}
    for name, shp in cfg.shapes().items():
        leaf = name.split(".")[-1]
        if leaf.endswith("_b"):
            t = torch.zeros(shp)
        elif leaf in ("ln1_w", "ln2_w", "lnf_w"):
            t = torch.ones(shp)
        else:
            t = torch.randn(shp, generator=g) * 0.02
        out[name] = t
    return out


class OptRanker:
    """Device-resident OPT-shape ranker: flat bf16 parameter buffer + forward."""

    def __init__(self, cfg: RankerConfig = RankerConfig(), seed: int | None = 0,
                 params: dict[str, torch.Tensor] | None = None, dev: torch.device | None = None):
        self.cfg = cfg
        self.dev = dev or _lib.device()
        self.total, self.offsets = layout(cfg)
        self.flat = torch.zeros(self.total, dtype=torch.bfloat16, device=self.dev)
        src = params if params is not None else init_params(cfg, 0 if seed is None else seed)
        self.load_state(src)

    def view(self, name: str) -> torch.Tensor:
        shp = self.cfg.shapes()[name]
        o = self.offsets[name]
        return self.flat[o:o + int(np.prod(shp))].view(shp)

    def load_state(self, params: dict[str, torch.Tensor]) -> None:
        for name in self.cfg.shapes():
            self.view(name).copy_(params[name].to(torch.bfloat16))

    def params_cpu_fp32(self) -> dict[str, torch.Tensor]:
        """The bf16 parameters upcast to fp32 on the CPU (what the oracle consumes)."""
        return {n: self.view(n).float().cpu() for n in self.cfg.shapes()}

    def workspace_bytes(self, B: int, S: int) -> int:
        c = self.cfg.c()
        return int(_lib.load().rs_ranker_workspace_size(ctypes.byref(c), B, S))

    def forward(self, ids: torch.Tensor, last_pos: torch.Tensor | None = None,
                out: torch.Tensor | None = None, score_out: torch.Tensor | None = None) -> torch.Tensor:
        """ids int32 [B, S] on the device -> g fp32 [B] (net output; higher = shorter).
        score_out (optional, fp32 [B]) receives -g, the scheduler's score."""
        if ids.dim() != 2:
            raise ValueError("ids must be [B, S]")
        B, S = ids.shape
        ids = ids.to(self.dev, torch.int32).contiguous()
        lp = None if last_pos is None else last_pos.to(self.dev, torch.int32).contiguous()
        g = out if out is not None else torch.empty(B, dtype=torch.float32, device=self.dev)
        lib = _lib.load()
        c = self.cfg.c()
        ws, wn = _lib.workspace.get(self.workspace_bytes(B, S), self.dev)
        _lib.check(lib.rs_ranker_forward(ctypes.byref(c), self.flat.data_ptr(), ids.data_ptr(),
                                         None if lp is None else lp.data_ptr(), B, S, g.data_ptr(),
                                         None if score_out is None else score_out.data_ptr(), ws, wn,
                                         _lib.stream_handle(self.dev)), "rs_ranker_forward")
        return g

    def features(self, ids: torch.Tensor, last_pos: torch.Tensor | None = None) -> torch.Tensor:
        """LN_f(h[last_pos]) fp32 [B, d]: the input of the classification head (§8f #4)."""
        if ids.dim() != 2:
            raise ValueError("ids must be [B, S]")
        B, S = ids.shape
        ids = ids.to(self.dev, torch.int32).contiguous()
        lp = None if last_pos is None else last_pos.to(self.dev, torch.int32).contiguous()
        g = torch.empty(B, dtype=torch.float32, device=self.dev)
        feat = torch.empty(B, self.cfg.d_model, dtype=torch.float32, device=self.dev)
        lib = _lib.load()
        c = self.cfg.c()
        ws, wn = _lib.workspace.get(self.workspace_bytes(B, S), self.dev)
        _lib.check(lib.rs_ranker_forward_ex(ctypes.byref(c), self.flat.data_ptr(), ids.data_ptr(), _lib.ptr(lp), B, S,
                                            g.data_ptr(), None, feat.data_ptr(), ws, wn, _lib.stream_handle(self.dev)),
                   "rs_ranker_forward_ex")
        return feat

    def forward_sharded(self, ids: torch.Tensor, last_pos: torch.Tensor | None = None, group=None) -> torch.Tensor:
        """Data-parallel scoring: this rank scores its contiguous shard of the
        global batch `ids` [B, S] and the fp32 outputs of all B prompts are all-gathered
        (NCCL) in prompt order. One rank: plain forward."""
        world, rank = dp.world_rank(group)
        lo, hi = dp.shard_range(ids.shape[0], world, rank)
        if hi > lo:
            g = self.forward(ids[lo:hi], None if last_pos is None else last_pos[lo:hi])
        else:
            g = torch.empty(0, dtype=torch.float32, device=ids.device)
        return dp.gather_scores(g, ids.shape[0], group)
