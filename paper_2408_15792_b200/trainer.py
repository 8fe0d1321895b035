"""ListMLE training of the OPT-shape ranker on B200s (A10/A11 of SURVEY §8a).

Reference: train_ranking (predictors.py:347-406): per minibatch list, order by bucketed
true length (stable), forward, list_mle_loss / n, list_mle_gradient / n, backward, Adam
(predictors.py:209-225). Here one optimizer step consumes many whole lists: each rank
accumulates the gradient of its lists with rs_ranker_grad (forward + fused ListMLE +
tcgen05 backward), the gradients are summed across data-parallel ranks with one NCCL
all-reduce of the flat fp32 buffer, and every rank applies the same fused Adam
(rs_adam_step, grad_scale = 1 / global lists) to its fp32 master copy. With one list
per step and one rank this is the reference's update sequence.
"""

from __future__ import annotations

import ctypes
import dataclasses

import torch
from . import _lib, dp
from .ranker import OptRanker


class RankerTrainer:
    def __init__(self, model: OptRanker, lr: float = 2e-5, betas=(0.9, 0.999), eps: float = 1e-8,
                 bucket_width: int = 10, lists_per_micro: int = 16, group=None):
        if bucket_width < 1:
            raise ValueError("bucket_width must be >= 1")
        self.model = model
        self.lr, self.betas, self.eps = float(lr), (float(betas[0]), float(betas[1])), float(eps)
        self.bucket_width = int(bucket_width)
        self.lists_per_micro = int(lists_per_micro)
        self.group = group
        dev = model.dev
        self.master = model.flat.float()
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)
        self.grad = torch.zeros_like(self.master)
        self.t = 0

    def _world(self) -> int:
        return dp.world_rank(self.group)[0]

    def accumulate(self, ids: torch.Tensor, lengths: torch.Tensor, list_len: int,
                   last_pos: torch.Tensor | None = None) -> torch.Tensor:
        """Add the gradient of sum_lists ListMLE/list_len for this rank's lists to .grad;
        returns the per-list losses (device tensor). last_pos (int32 [n], optional) is
        each prompt's last real token (the score is read there, as in forward)."""
        n_prompts, S = ids.shape
        if n_prompts % list_len:
            raise ValueError("ids rows must be whole lists")
        n_lists = n_prompts // list_len
        dev = self.model.dev
        ids = ids.to(dev, torch.int32).contiguous()
        lengths = lengths.to(dev, torch.int32).contiguous().view(-1)
        lp = None if last_pos is None else last_pos.to(dev, torch.int32).contiguous().view(-1)
        loss = torch.empty(n_lists, dtype=torch.float32, device=dev)
        lib = _lib.load()
        c = self.model.cfg.c()
        mb = min(self.lists_per_micro, n_lists)
        need = lib.rs_ranker_grad_workspace_size(ctypes.byref(c), mb, list_len, S)
        ws, wn = _lib.workspace.get(need, dev)
        _lib.check(lib.rs_ranker_grad(ctypes.byref(c), self.model.flat.data_ptr(), self.grad.data_ptr(),
                                      ids.data_ptr(), _lib.ptr(lp), lengths.data_ptr(), n_lists, list_len, S, self.bucket_width,
                                      mb, loss.data_ptr(), ws, wn, _lib.stream_handle(dev)), "rs_ranker_grad")
        return loss

    def apply(self, total_lists: int) -> None:
        """All-reduce the accumulated gradient across ranks (NCCL) and take one Adam step."""
        dp.allreduce_sum_(self.grad, self.group)
        self.apply_local(total_lists)

    def apply_local(self, total_lists: int) -> None:
        """One Adam step on .grad as it stands (already summed over ranks), scaled by
        1 / total_lists; zeroes .grad."""
        self.t += 1
        _lib.check(_lib.load().rs_adam_step(self.master.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                                            self.grad.data_ptr(), self.model.flat.data_ptr(), self.master.numel(),
                                            self.lr, self.betas[0], self.betas[1], self.eps, self.t,
                                            1.0 / float(total_lists), _lib.stream_handle(self.model.dev)),
                   "rs_adam_step")

    # ---- checkpoint / resume ------------------------------------------------------------
    def state_dict(self) -> dict:
        """Everything the next step depends on: the fp32 master weights, both Adam moments,
        the step count and hyper-parameters (the bf16 working copy is re-derived)."""
        return {"format": "rsb200-ranker-trainer", "version": 1, "t": self.t, "lr": self.lr,
                "betas": list(self.betas), "eps": self.eps, "bucket_width": self.bucket_width,
                "config": dataclasses.asdict(self.model.cfg),
                "master": self.master.cpu(), "m": self.m.cpu(), "v": self.v.cpu(),
                "params_bf16": self.model.flat.cpu()}

    def load_state_dict(self, sd: dict) -> None:
        if sd.get("format") != "rsb200-ranker-trainer" or sd.get("version") != 1:
            raise ValueError("not a ranker-trainer checkpoint")
        if sd["config"] != dataclasses.asdict(self.model.cfg):
            raise ValueError("checkpoint was written for a different ranker config")
        if sd["master"].numel() != self.master.numel():
            raise ValueError("checkpoint parameter count mismatch")
        self.t, self.lr, self.eps = int(sd["t"]), float(sd["lr"]), float(sd["eps"])
        self.betas, self.bucket_width = (float(sd["betas"][0]), float(sd["betas"][1])), int(sd["bucket_width"])
        self.master.copy_(sd["master"])
        self.m.copy_(sd["m"])
        self.v.copy_(sd["v"])
        self.model.flat.copy_(sd["params_bf16"])
        self.grad.zero_()

    def save_checkpoint(self, path: str) -> None:
        torch.save(self.state_dict(), path)

    def load_checkpoint(self, path: str) -> None:
        self.load_state_dict(torch.load(path, map_location="cpu", weights_only=True))

    def step(self, ids: torch.Tensor, lengths: torch.Tensor, list_len: int, total_lists: int | None = None,
             last_pos: torch.Tensor | None = None):
        loss = self.accumulate(ids, lengths, list_len, last_pos)
        n_lists = ids.shape[0] // list_len
        self.apply(total_lists if total_lists is not None else n_lists * self._world())
        return loss


def classifier_logits(model: OptRanker, W: torch.Tensor, b: torch.Tensor, ids: torch.Tensor,
                      last_pos: torch.Tensor | None = None) -> torch.Tensor:
    """logits [B, C] = LN_f(h_last) W^T + b (rs_ranker_forward_ex features + rs_cls_logits)."""
    feat = model.features(ids, last_pos)
    B, d = feat.shape
    C = W.shape[0]
    W = W.to(model.dev, torch.float32).contiguous()
    b = b.to(model.dev, torch.float32).contiguous()
    out = torch.empty(B, C, dtype=torch.float32, device=model.dev)
    _lib.check(_lib.load().rs_cls_logits(feat.data_ptr(), W.data_ptr(), b.data_ptr(), B, d, C, out.data_ptr(),
                                         _lib.stream_handle(model.dev)), "rs_cls_logits")
    return out


class ClassifierTrainer:
    """The bucketed-classification baseline on the same backbone (§8f #4; reference:
    train_classifier, predictors.py:409-479): a C-way linear head on LN_f(h_last),
    softmax cross-entropy, Adam on the backbone and the head. accumulate() adds the
    gradient of the summed per-prompt nll (rs_ranker_grad_cls); apply() all-reduces and
    steps with grad_scale = 1 / prompts (the reference's batch mean)."""

    def __init__(self, model: OptRanker, n_classes: int, lr: float = 2e-5, betas=(0.9, 0.999), eps: float = 1e-8,
                 prompts_per_micro: int = 256, group=None):
        if n_classes < 2:
            raise ValueError("classification needs at least 2 buckets")
        self.model, self.n_classes = model, int(n_classes)
        self.lr, self.betas, self.eps = float(lr), (float(betas[0]), float(betas[1])), float(eps)
        self.prompts_per_micro, self.group = int(prompts_per_micro), group
        dev, d = model.dev, model.cfg.d_model
        self.master = model.flat.float()
        self.m, self.v, self.grad = (torch.zeros_like(self.master) for _ in range(3))
        # head: W [C, d] then b [C], fp32, zero-initialised like the reference (predictors.py:438-439)
        self.head = torch.zeros(self.n_classes * d + self.n_classes, dtype=torch.float32, device=dev)
        self.hm, self.hv, self.hgrad = (torch.zeros_like(self.head) for _ in range(3))
        self._head_bf16 = torch.empty(self.head.numel(), dtype=torch.bfloat16, device=dev)  # Adam's bf16 copy (unused)
        self.t = 0

    @property
    def W(self) -> torch.Tensor:
        return self.head[:self.n_classes * self.model.cfg.d_model].view(self.n_classes, -1)

    @property
    def b(self) -> torch.Tensor:
        return self.head[self.n_classes * self.model.cfg.d_model:]

    def logits(self, ids: torch.Tensor, last_pos: torch.Tensor | None = None) -> torch.Tensor:
        return classifier_logits(self.model, self.W, self.b, ids, last_pos)

    def accumulate(self, ids: torch.Tensor, labels: torch.Tensor, last_pos: torch.Tensor | None = None):
        n, S = ids.shape
        dev = self.model.dev
        labels = labels.to(dev, torch.int32).contiguous().view(-1)
        if labels.numel() != n or int(labels.min()) < 0 or int(labels.max()) >= self.n_classes:
            raise ValueError("labels must be one class in [0, n_classes) per prompt")
        ids = ids.to(dev, torch.int32).contiguous()
        lp = None if last_pos is None else last_pos.to(dev, torch.int32).contiguous().view(-1)
        loss = torch.empty(n, dtype=torch.float32, device=dev)
        lib = _lib.load()
        c = self.model.cfg.c()
        mb = min(self.prompts_per_micro, n)
        need = lib.rs_ranker_grad_cls_workspace_size(ctypes.byref(c), mb, S, self.n_classes)
        ws, wn = _lib.workspace.get(need, dev)
        _lib.check(lib.rs_ranker_grad_cls(ctypes.byref(c), self.model.flat.data_ptr(), self.grad.data_ptr(),
                                          ids.data_ptr(), _lib.ptr(lp), labels.data_ptr(), n, S, self.n_classes,
                                          self.W.data_ptr(), self.b.data_ptr(), self.hgrad.data_ptr(), mb,
                                          loss.data_ptr(), ws, wn, _lib.stream_handle(dev)), "rs_ranker_grad_cls")
        return loss

    def apply(self, total_prompts: int) -> None:
        dp.allreduce_sum_(self.grad, self.group)
        dp.allreduce_sum_(self.hgrad, self.group)
        self.t += 1
        lib, st = _lib.load(), _lib.stream_handle(self.model.dev)
        for master, m, v, g, pb in ((self.master, self.m, self.v, self.grad, self.model.flat),
                                    (self.head, self.hm, self.hv, self.hgrad, self._head_bf16)):
            _lib.check(lib.rs_adam_step(master.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), pb.data_ptr(),
                                        master.numel(), self.lr, self.betas[0], self.betas[1], self.eps, self.t,
                                        1.0 / float(total_prompts), st), "rs_adam_step")
