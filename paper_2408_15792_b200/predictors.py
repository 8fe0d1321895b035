"""Scorer plugin for the OPT-shape ranker (drop-in for the ranksched Scorer protocol).

The reference Scorer contract (predictors.py:35-51): class attributes `kind`,
`length_calibrated`, `warmup_tokens`, `charges_predictor`; `score_batch(requests,
seed) -> list[float | None]`; `to_dict()` with a `kind` key. RankingModelScorer
(predictors.py:228-259) negates the net output so that the ascending sort puts
predicted-short requests first; OptRankerScorer keeps that orientation with the
paper's OPT backbone in place of the 24-feature _Net.

Serialization (predictors.py:486-527 uses JSON for the tiny linear model): 125M bf16
parameters do not fit the JSON payload, so save_scorer writes the JSON header (same
`format`/`version` keys, kind "opt-ranker") plus a raw little-endian bf16 sidecar
`<path>.bin` whose sha256 the header records.
"""

from __future__ import annotations

import dataclasses
import hashlib
import math
import json
import pathlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .ranker import OptRanker, RankerConfig
from .workload import prompt_token_ids, prompt_token_ids_device

_SCORER_FORMAT = "ranksched-scorer"
_SCORER_VERSION = 1


class OptRankerScorer:
    """OPT-125M-shape ranker; score = -(net output), not length calibrated."""

    kind = "opt-ranker"
    length_calibrated = False
    warmup_tokens = 0
    charges_predictor = True

    def __init__(self, model: OptRanker | None = None, seq_len: int = 128, cfg: RankerConfig | None = None,
                 seed: int = 0, device_tokenizer: bool | str = "auto"):
        self.model = model if model is not None else OptRanker(cfg or RankerConfig(), seed=seed)
        self.seq_len = int(seq_len)
        self.weights_path: str | None = None
        # prompts -> ids (identical either way): True = on the device (rs_tokenize; ASCII
        # prompts only, others raise); False = the host map; "auto" = the device, with
        # the host map patching in the rows of prompts that need Unicode-aware splitting
        if device_tokenizer not in (True, False, "auto"):
            raise ValueError("device_tokenizer must be True, False or 'auto'")
        self.device_tokenizer = device_tokenizer

    def encode(self, requests) -> tuple[torch.Tensor, torch.Tensor]:
        """Prompts -> (ids int32 [n, S], last_pos int32 [n]) in pinned host memory."""
        n = len(requests)
        ids = torch.empty((n, self.seq_len), dtype=torch.int32).pin_memory()
        last = torch.empty(n, dtype=torch.int32).pin_memory()
        ids_np, last_np = ids.numpy(), last.numpy()
        for k, r in enumerate(requests):
            ids_np[k], last_np[k] = prompt_token_ids(getattr(r, "prompt", "") or "", self.seq_len,
                                                     self.model.cfg.vocab)
        return ids, last

    def raw_outputs(self, requests) -> np.ndarray:
        if not requests:
            return np.zeros(0)
        dev = self.model.dev
        if self.device_tokenizer:
            ids, last = prompt_token_ids_device([getattr(r, "prompt", "") or "" for r in requests], self.seq_len,
                                                self.model.cfg.vocab, device=dev,
                                                host_fallback=self.device_tokenizer == "auto")
            g = self.model.forward(ids, last)
        else:
            ids, last = self.encode(requests)
            g = self.model.forward(ids.to(dev, non_blocking=True), last.to(dev, non_blocking=True))
        return g.double().cpu().numpy()

    def score_batch(self, requests, seed) -> list[float | None]:
        return [-float(v) for v in self.raw_outputs(list(requests))]

    def to_dict(self) -> dict:
        """JSON-able description (the reference engine hashes it into the run config,
        engine.py:366). `weights_sha256` hashes the parameters in memory, so it tracks the
        current weights whether or not they were saved; `weights` is the sidecar written
        by save_scorer() (absolute path), or None before that."""
        return {"kind": self.kind, "config": dataclasses.asdict(self.model.cfg), "seq_len": self.seq_len,
                "weights": self.weights_path, "weights_sha256": _sha256_params(self.model.flat)}


def _sha256_params(flat: torch.Tensor) -> str:
    """sha256 of the raw little-endian bf16 parameter bytes (== the sidecar file's)."""
    return hashlib.sha256(flat.view(torch.int16).cpu().numpy().tobytes()).hexdigest()


def _sha256_file(path) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 24), b""):
            h.update(chunk)
    return h.hexdigest()


def save_scorer(scorer, path: str) -> None:
    """JSON header at `path` + raw bf16 parameters at `path + '.bin'`. The header names
    the sidecar relative to its own directory (load_scorer resolves it there)."""
    p = pathlib.Path(path)
    weights = p.with_name(p.name + ".bin")
    scorer.model.flat.view(torch.int16).cpu().numpy().tofile(weights)
    scorer.weights_path = str(weights.resolve())
    payload = {"format": _SCORER_FORMAT, "version": _SCORER_VERSION}
    payload.update(scorer.to_dict())
    payload["weights"] = weights.name
    p.write_text(json.dumps(payload) + "\n", encoding="utf-8")


def scorer_from_dict(obj: dict, base_dir: str | None = None):
    """`kind == "opt-ranker"` -> OptRankerScorer, "opt-classifier" -> OptClassifierScorer;
    other kinds belong to the reference
    (ranksched.predictors.scorer_from_dict; install() chains the two). A relative
    `weights` path is resolved against `base_dir` (load_scorer: the header's directory)."""
    kind = obj.get("kind")
    if kind not in (OptRankerScorer.kind, "opt-classifier"):
        raise ValueError(f"unknown scorer kind {kind!r}")
    if not obj.get("weights"):
        raise ValueError(f"{kind} scorer dict has no weights file: save it with save_scorer() first")
    cfg = RankerConfig(**obj["config"])
    model = OptRanker(cfg, seed=None)
    weights = pathlib.Path(obj["weights"])
    if not weights.is_absolute() and base_dir is not None:
        weights = pathlib.Path(base_dir) / weights
    weights = str(weights)
    if obj.get("weights_sha256") and _sha256_file(weights) != obj["weights_sha256"]:
        raise ValueError(f"{weights}: checksum mismatch")
    raw = np.fromfile(weights, dtype=np.int16)
    if raw.size != model.flat.numel():
        raise ValueError(f"{weights}: {raw.size} parameters, expected {model.flat.numel()}")
    model.flat.view(torch.int16).copy_(torch.from_numpy(raw))
    if kind == "opt-classifier":
        s = OptClassifierScorer(model, torch.tensor(obj["head_weights"], dtype=torch.float32),
                                torch.tensor(obj["head_bias"], dtype=torch.float32), obj["bucket_size"],
                                seq_len=obj.get("seq_len", 128))
    else:
        s = OptRankerScorer(model, seq_len=obj.get("seq_len", 128))
    s.weights_path = str(pathlib.Path(weights).resolve())
    return s


def load_scorer(path: str):
    with open(path, "r", encoding="utf-8") as fh:
        obj = json.load(fh)
    if obj.get("format") != _SCORER_FORMAT:
        raise ValueError(f"{path}: not a scorer file")
    if obj.get("version") != _SCORER_VERSION:
        raise ValueError(f"{path}: unsupported scorer version {obj.get('version')}")
    return scorer_from_dict(obj, base_dir=str(pathlib.Path(path).parent))


@dataclass(frozen=True)
class TrainConfig:
    """The reference's TrainConfig fields (predictors.py:308-318) plus the ranker shape.

    Defaults follow the paper's recipe for the OPT predictor: Adam lr
    2e-5, betas (0.9, 0.999), list (batch) size 32, bucket width 10, 5 epochs.
    `lists_per_step` batches that many independent lists per optimizer step (the
    reference does one list per step; with lists_per_step=1 the update sequence is
    the reference's)."""

    epochs: int = 5
    batch_size: int = 32
    learning_rate: float = 2e-5
    betas: tuple[float, float] = (0.9, 0.999)
    bucket_width: int = 10
    hidden: int = 0
    checkpoint_every: int = 20
    eval_fraction: float = 0.2
    seed: int = 0
    seq_len: int = 128
    lists_per_step: int = 1
    lists_per_micro: int = 16
    ranker: RankerConfig = RankerConfig()


@dataclass
class TrainResult:
    scorer: object
    report: dict = field(default_factory=dict)


def _encode(requests, seq_len: int, vocab: int):
    ids = np.empty((len(requests), seq_len), dtype=np.int32)
    last = np.empty(len(requests), dtype=np.int32)
    for k, r in enumerate(requests):
        ids[k], last[k] = prompt_token_ids(getattr(r, "prompt", "") or "", seq_len, vocab)
    return ids, last


def _split_requests(reqs, cfg: TrainConfig, eval_trace):
    """Train / eval split of _split_features (predictors.py:327-340)."""
    if eval_trace is not None:
        return reqs, list(eval_trace)
    rng0 = np.random.default_rng(cfg.seed)
    idx = rng0.permutation(len(reqs))
    n_eval = max(1, int(round(cfg.eval_fraction * len(reqs))))
    if n_eval >= len(reqs):
        raise ValueError("trace too small to split for evaluation")
    return [reqs[i] for i in idx[n_eval:]], [reqs[i] for i in idx[:n_eval]]


def train_ranking(trace, cfg: TrainConfig = TrainConfig(), eval_trace=None, model: OptRanker | None = None,
                  group=None) -> TrainResult:
    """ListMLE training of the OPT-shape ranker (reference: train_ranking,
    predictors.py:347-406, same split, shuffling, list construction, checkpoints and
    report keys).

    Every minibatch of `batch_size` requests is one ranked list whose target order is
    the stable argsort of bucketed true lengths (predictors.py:379-381); the list's
    ListMLE loss / n and its gradient come from the fused device pass (rs_ranker_grad,
    forward + K6 + tcgen05 backward). `lists_per_step` consecutive lists share one Adam
    step (gradient = mean over lists); 1 reproduces the reference's one-list-per-step
    sequence. Under torch.distributed the lists of a step are split across ranks and
    the gradient is all-reduced (NCCL) before the replicated Adam step.
    """
    from . import dp
    from .ranking import kendall_tau_b
    from .trainer import RankerTrainer

    reqs = list(trace)
    if len(reqs) < 4:
        raise ValueError("need at least 4 requests to train")
    if cfg.bucket_width < 1:
        raise ValueError("bucket_width must be >= 1")
    if cfg.lists_per_step < 1:
        raise ValueError("lists_per_step must be >= 1")
    tr_reqs, ev_reqs = _split_requests(reqs, cfg, eval_trace)
    rc = cfg.ranker
    if model is None:
        model = OptRanker(rc, seed=cfg.seed)
    dev = model.dev
    ids_np, last_np = _encode(tr_reqs, cfg.seq_len, rc.vocab)
    eids_np, elast_np = _encode(ev_reqs, cfg.seq_len, rc.vocab)
    y = np.array([r.true_output_tokens for r in tr_reqs], dtype=np.int64)
    ye = np.array([r.true_output_tokens for r in ev_reqs], dtype=np.int64)
    ids = torch.from_numpy(ids_np).to(dev)
    last = torch.from_numpy(last_np).to(dev)
    yd = torch.from_numpy(y.astype(np.int32)).to(dev)
    eids = torch.from_numpy(eids_np).to(dev)
    elast = torch.from_numpy(elast_np).to(dev)

    world, rank = dp.world_rank(group)
    trainer = RankerTrainer(model, lr=cfg.learning_rate, betas=cfg.betas, bucket_width=cfg.bucket_width,
                            lists_per_micro=cfg.lists_per_micro, group=group)

    def eval_tau() -> float:
        g = model.forward(eids, elast)
        return kendall_tau_b(-g, ye).tau

    rng = np.random.default_rng(cfg.seed + 1)
    step = 0
    window: list[torch.Tensor] = []
    checkpoints: list[dict] = []
    for _epoch in range(cfg.epochs):
        order = rng.permutation(len(y))
        lists = [order[s:s + cfg.batch_size] for s in range(0, len(order), cfg.batch_size)]
        lists = [b for b in lists if len(b) >= 2]
        for g0 in range(0, len(lists), cfg.lists_per_step):
            grp = lists[g0:g0 + cfg.lists_per_step]
            losses = []
            for b in dp.shard_lists(grp, world, rank):
                bi = torch.from_numpy(b).to(dev)
                losses.append(trainer.accumulate(ids[bi], yd[bi], len(b), last[bi]))
            trainer.apply(len(grp))
            step_loss = torch.cat(losses).sum() if losses else torch.zeros((), device=dev)
            dp.allreduce_sum_(step_loss, group)
            window.append(step_loss / len(grp))
            step += 1
            if step % cfg.checkpoint_every == 0:
                checkpoints.append({"step": step, "train_loss": float(torch.stack(window).mean().item()),
                                    "eval_tau": eval_tau()})
                window = []
    final_tau = eval_tau()
    scorer = OptRankerScorer(model, seq_len=cfg.seq_len)
    report = {"kind": "ranking", "steps": step, "checkpoints": checkpoints, "eval_tau": final_tau,
              "n_train": len(y), "n_eval": len(ye)}
    return TrainResult(scorer, report)


class OptClassifierScorer:
    """The bucketed-classification baseline on the OPT backbone (reference:
    ClassifierScorer, predictors.py:262-300): argmax over C length buckets of a linear head
    (W [C, d], b [C], fp32) on LN_f(h_last); the score is the bucket's midpoint in tokens
    (length calibrated)."""

    kind = "opt-classifier"
    length_calibrated = True
    warmup_tokens = 0
    charges_predictor = True

    def __init__(self, model: OptRanker, weights: torch.Tensor, bias: torch.Tensor, bucket_size: int,
                 seq_len: int = 128):
        self.model = model
        self.weights = weights.to(model.dev, torch.float32).contiguous()
        self.bias = bias.to(model.dev, torch.float32).contiguous()
        self.bucket_size = int(bucket_size)
        self.seq_len = int(seq_len)
        self.weights_path: str | None = None

    @property
    def n_buckets(self) -> int:
        return int(self.bias.numel())

    def predict_buckets(self, requests) -> np.ndarray:
        from .trainer import classifier_logits
        ids_np, last_np = _encode(list(requests), self.seq_len, self.model.cfg.vocab)
        dev = self.model.dev
        lg = classifier_logits(self.model, self.weights, self.bias, torch.from_numpy(ids_np).to(dev),
                               torch.from_numpy(last_np).to(dev))
        return lg.argmax(dim=1).cpu().numpy()

    def score_batch(self, requests, seed) -> list[float | None]:
        reqs = list(requests)
        if not reqs:
            return []
        return [float(b * self.bucket_size + self.bucket_size / 2.0) for b in self.predict_buckets(reqs)]

    def to_dict(self) -> dict:
        return {"kind": self.kind, "config": dataclasses.asdict(self.model.cfg), "seq_len": self.seq_len,
                "bucket_size": self.bucket_size, "head_weights": self.weights.cpu().tolist(),
                "head_bias": self.bias.cpu().tolist(), "weights": self.weights_path,
                "weights_sha256": _sha256_params(self.model.flat)}


def train_classifier(trace, cfg: TrainConfig = TrainConfig(), n_buckets: int | None = 10,
                     bucket_size: int | None = None, eval_trace=None, model: OptRanker | None = None,
                     group=None) -> TrainResult:
    """Bucketed classification on the OPT backbone (reference: train_classifier,
    predictors.py:409-479 — same bucketing rules, split, per-epoch permutation, minibatches
    of batch_size, Adam; report keys kind/steps/n_buckets/bucket_size/accuracy/eval_tau/
    n_train/n_eval). Each minibatch is one optimizer step whose gradient is the batch mean
    of the cross-entropy (rs_ranker_grad_cls); under torch.distributed the batch is split
    across ranks and the gradients all-reduced."""
    from . import dp
    from .ranking import kendall_tau_b
    from .trainer import ClassifierTrainer

    reqs = list(trace)
    if len(reqs) < 4:
        raise ValueError("need at least 4 requests to train")
    tr_reqs, ev_reqs = _split_requests(reqs, cfg, eval_trace)
    y = np.array([r.true_output_tokens for r in tr_reqs], dtype=np.int64)
    ye = np.array([r.true_output_tokens for r in ev_reqs], dtype=np.int64)
    max_len = int(max(y.max(), ye.max()))
    if bucket_size is None:
        if n_buckets is None:
            raise ValueError("give n_buckets or bucket_size")
        bucket_size = max(1, math.ceil(max_len / n_buckets))
    if n_buckets is None:
        n_buckets = max_len // bucket_size + 1
    if n_buckets < 2:
        raise ValueError("classification needs at least 2 buckets")
    labels = np.minimum(y // bucket_size, n_buckets - 1)
    labels_e = np.minimum(ye // bucket_size, n_buckets - 1)
    rc = cfg.ranker
    if model is None:
        model = OptRanker(rc, seed=cfg.seed)
    dev = model.dev
    ids_np, last_np = _encode(tr_reqs, cfg.seq_len, rc.vocab)
    eids_np, elast_np = _encode(ev_reqs, cfg.seq_len, rc.vocab)
    ids, last = torch.from_numpy(ids_np).to(dev), torch.from_numpy(last_np).to(dev)
    lab = torch.from_numpy(labels.astype(np.int32)).to(dev)
    trainer = ClassifierTrainer(model, n_buckets, lr=cfg.learning_rate, betas=cfg.betas, group=group)
    world, rank = dp.world_rank(group)
    rng = np.random.default_rng(cfg.seed + 1)
    step = 0
    for _epoch in range(cfg.epochs):
        order = rng.permutation(len(y))
        for start in range(0, len(order), cfg.batch_size):
            batch = order[start:start + cfg.batch_size]
            if len(batch) == 0:
                continue
            lo, hi = dp.shard_range(len(batch), world, rank)
            if hi > lo:
                bi = torch.from_numpy(batch[lo:hi]).to(dev)
                trainer.accumulate(ids[bi], lab[bi], last[bi])
            trainer.apply(len(batch))
            step += 1
    scorer = OptClassifierScorer(model, trainer.W.detach().clone(), trainer.b.detach().clone(), bucket_size,
                                 seq_len=cfg.seq_len)
    lg = trainer.logits(torch.from_numpy(eids_np).to(dev), torch.from_numpy(elast_np).to(dev))
    pred_e = lg.argmax(dim=1).cpu().numpy()
    midpoints = pred_e * bucket_size + bucket_size / 2.0
    report = {"kind": "classifier", "steps": step, "n_buckets": int(n_buckets), "bucket_size": int(bucket_size),
              "accuracy": float(np.mean(pred_e == labels_e)), "eval_tau": kendall_tau_b(midpoints, ye).tau,
              "n_train": len(y), "n_eval": len(ye)}
    return TrainResult(scorer, report)
