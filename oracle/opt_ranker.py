"""CPU fp32 restatement of the OPT-shape ranker — TEST INFRASTRUCTURE ONLY (checker).

The reference package has no backbone (SPEC.md:12 puts the OPT predictor out of
scope); the paper's predictor is "a small OPT model ... a linear layer to map the
hidden states of the last layer to a floating-point number as a score"
(PAPER.md:195-201). This is a plain torch fp32 statement of HF OPT-125M semantics
(learned positions with offset 2, pre-LN, q scaled by 1/sqrt(head_dim), causal
softmax, ReLU FFN, final LayerNorm) + Linear(d, 1) on the last prompt token, taking
the same parameter dict the B200 ranker holds (bf16 values upcast to fp32). It is
pinned to transformers' OPTModel by tests/golden/make_opt_golden.py.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F


def _ln(x, w, b):
    return F.layer_norm(x, (x.shape[-1],), w, b, eps=1e-5)


def hidden_states_grad(params, cfg, ids) -> torch.Tensor:
    """hidden_states with autograd (the fp32 training reference / the CPU train baseline)."""
    ids = torch.as_tensor(np.asarray(ids), dtype=torch.long, device=params["tok_emb"].device)
    B, S = ids.shape
    d, H = cfg.d_model, cfg.n_heads
    hd = d // H
    dev = params["tok_emb"].device
    h = params["tok_emb"][ids] + params["pos_emb"][torch.arange(S, device=dev) + 2][None]
    mask = torch.full((S, S), float("-inf"), device=dev).triu(1)
    for layer in range(cfg.n_layers):
        p = {k.split(".")[-1]: v for k, v in params.items() if k.startswith(f"layers.{layer}.")}
        x = _ln(h, p["ln1_w"], p["ln1_b"])
        qkv = x @ p["qkv_w"].t() + p["qkv_b"]
        q, k, v = qkv.split(d, dim=-1)
        q = q.view(B, S, H, hd).transpose(1, 2) * (hd ** -0.5)
        k = k.view(B, S, H, hd).transpose(1, 2)
        v = v.view(B, S, H, hd).transpose(1, 2)
        att = torch.softmax(q @ k.transpose(-1, -2) + mask, dim=-1) @ v
        att = att.transpose(1, 2).reshape(B, S, d)
        h = h + att @ p["out_w"].t() + p["out_b"]
        x = _ln(h, p["ln2_w"], p["ln2_b"])
        f = x @ p["fc1_w"].t() + p["fc1_b"]
        f = torch.relu(f) if cfg.activation == 0 else F.gelu(f, approximate="tanh")
        h = h + f @ p["fc2_w"].t() + p["fc2_b"]
    return h


hidden_states = torch.no_grad()(hidden_states_grad)


def forward_grad(params, cfg, ids, last_pos=None) -> torch.Tensor:
    """g [B] fp32 = head_w . LN_f(h[b, last_pos[b]]) + head_b (higher = shorter), with autograd."""
    h = hidden_states_grad(params, cfg, ids)
    B, S = h.shape[:2]
    lp = torch.full((B,), S - 1, dtype=torch.long) if last_pos is None else torch.as_tensor(last_pos).long()
    last = h[torch.arange(B), lp.to(h.device)]
    x = _ln(last, params["lnf_w"], params["lnf_b"])
    return x @ params["head_w"] + params["head_b"][0]


forward = torch.no_grad()(forward_grad)


def listmle_torch(g, lengths, width=10):
    """sum over lists of list_mle_loss(g_list, stable argsort(len // width)) / n
    (ranking.py:86-99, predictors.py:380-383) in torch (autograd-able)."""
    total = 0.0
    for gl, ll in zip(g, lengths):
        order = torch.from_numpy(np.argsort(np.asarray(ll) // width, kind="stable")).to(gl.device)
        t = gl[order]
        lse = torch.logcumsumexp(t.flip(0), 0).flip(0)
        total = total + (lse - t).sum() / len(gl)
    return total
