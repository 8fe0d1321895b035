"""The reference's own ranker on the B200: standardised 24-feature linear / MLP net trained
with ListMLE (A2/A3 of SURVEY §8a) — the parity bridge for BASELINE configs[0].

Reference: _Standardizer (predictors.py:159-172), _Net (:175-206), _Adam (:209-225),
RankingModelScorer (:228-259), TrainConfig (:308-318), _split_features (:327-340),
train_ranking (:347-406). Same split, shuffles, list construction, initialisation,
checkpoints, report keys and to_dict() format; the arithmetic (standardisation, forward,
stable bucket order, ListMLE, backward, Adam) runs in float64 kernels of librsb200
(rs_standardizer_fit, rs_linear_forward, rs_linear_train_step). Features are the
reference's featurize (workload.featurize, host string work) read from Request.features.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .workload import featurize


@dataclass(frozen=True)
class FeatureTrainConfig:
    """The reference TrainConfig (predictors.py:308-318), same defaults."""

    epochs: int = 5
    batch_size: int = 32
    learning_rate: float = 1e-2
    betas: tuple[float, float] = (0.9, 0.999)
    bucket_width: int = 10
    hidden: int = 0
    checkpoint_every: int = 20
    eval_fraction: float = 0.2
    seed: int = 0


def _features(requests) -> np.ndarray:
    rows = []
    for r in requests:
        f = getattr(r, "features", None)
        rows.append(f if f is not None else featurize(getattr(r, "prompt", "") or ""))
    return np.stack(rows).astype(np.float64, copy=False) if rows else np.zeros((0, 24))


def init_params(dim: int, hidden: int, rng: np.random.Generator) -> list[np.ndarray]:
    """_Net.init (predictors.py:184-190): zeros for the linear model, N(0, 1/dim) /
    N(0, 1/hidden) weights and zero biases for the MLP — same draws."""
    if hidden <= 0:
        return [np.zeros(dim), np.zeros(1)]
    w1 = rng.normal(0.0, 1.0 / math.sqrt(dim), size=(dim, hidden))
    w2 = rng.normal(0.0, 1.0 / math.sqrt(hidden), size=hidden)
    return [w1, np.zeros(hidden), w2, np.zeros(1)]


class RankingModelScorer:
    """Drop-in for the reference RankingModelScorer (kind "ranking-model"): score =
    -net(standardise(features)), not length calibrated, charges the predictor."""

    kind = "ranking-model"
    length_calibrated = False
    warmup_tokens = 0
    charges_predictor = True

    def __init__(self, params: list, hidden: int, mean, std, dev: torch.device | None = None):
        self.dev = dev or _lib.device()
        self.hidden = int(hidden)
        self.shapes = [np.shape(p) for p in params]
        flat = np.concatenate([np.asarray(p, dtype=np.float64).ravel() for p in params])
        self.dim = int(np.asarray(mean).size)
        if flat.size != _lib.load().rs_linear_n_params(self.dim, self.hidden):
            raise ValueError("params do not match (n_features, hidden)")
        self.flat = torch.from_numpy(flat).to(self.dev)
        self.mean = torch.as_tensor(np.asarray(mean, dtype=np.float64)).to(self.dev)
        self.std = torch.as_tensor(np.asarray(std, dtype=np.float64)).to(self.dev)

    @property
    def params(self) -> list[np.ndarray]:
        flat = self.flat.cpu().numpy()
        out, o = [], 0
        for shp in self.shapes:
            k = int(np.prod(shp)) if shp else 1
            out.append(flat[o:o + k].reshape(shp))
            o += k
        return out

    def raw_outputs_features(self, X: np.ndarray | torch.Tensor) -> torch.Tensor:
        X = torch.as_tensor(X, dtype=torch.float64).to(self.dev).contiguous()
        n = X.shape[0]
        out = torch.empty(n, dtype=torch.float64, device=self.dev)
        _lib.check(_lib.load().rs_linear_forward(X.data_ptr(), n, self.dim, self.mean.data_ptr(), self.std.data_ptr(),
                                                 self.hidden, self.flat.data_ptr(), out.data_ptr(),
                                                 _lib.stream_handle(self.dev)), "rs_linear_forward")
        return out

    def raw_outputs(self, requests) -> np.ndarray:
        reqs = list(requests)
        if not reqs:
            return np.zeros(0)
        return self.raw_outputs_features(_features(reqs)).cpu().numpy()

    def score_batch(self, requests, seed) -> list[float | None]:
        return [-float(v) for v in self.raw_outputs(requests)]

    def to_dict(self) -> dict:
        return {"kind": self.kind, "hidden": self.hidden, "params": [p.tolist() for p in self.params],
                "feat_mean": self.mean.cpu().tolist(), "feat_std": self.std.cpu().tolist()}

    @classmethod
    def from_dict(cls, obj: dict) -> "RankingModelScorer":
        return cls([np.array(p) for p in obj["params"]], obj["hidden"], obj["feat_mean"], obj["feat_std"])


def train_ranking_features(trace, cfg: FeatureTrainConfig = FeatureTrainConfig(), eval_trace=None):
    """train_ranking (predictors.py:347-406) on the device: every minibatch list is one
    rs_linear_train_step (gather, forward, stable bucket order, ListMLE / n, backward,
    Adam); checkpoints every `checkpoint_every` steps with eval tau (kendall_tau_b on the
    device). Returns predictors.TrainResult(RankingModelScorer, report)."""
    from .predictors import TrainResult
    from .ranking import kendall_tau_b

    reqs = list(trace)
    if len(reqs) < 4:
        raise ValueError("need at least 4 requests to train")
    if cfg.bucket_width < 1:
        raise ValueError("bucket_width must be >= 1")
    dev = _lib.device()
    lib = _lib.load()
    st = _lib.stream_handle(dev)
    X = _features(reqs)
    y = np.array([r.true_output_tokens for r in reqs], dtype=np.int64)
    if eval_trace is not None:
        ev = list(eval_trace)
        Xe, ye = _features(ev), np.array([r.true_output_tokens for r in ev], dtype=np.int64)
    else:  # _split_features (predictors.py:327-340)
        idx = np.random.default_rng(cfg.seed).permutation(len(y))
        n_eval = max(1, int(round(cfg.eval_fraction * len(y))))
        if n_eval >= len(y):
            raise ValueError("trace too small to split for evaluation")
        X, y, Xe, ye = X[idx[n_eval:]], y[idx[n_eval:]], X[idx[:n_eval]], y[idx[:n_eval]]
    D = X.shape[1]
    Xd = torch.from_numpy(np.ascontiguousarray(X)).to(dev)
    Xed = torch.from_numpy(np.ascontiguousarray(Xe)).to(dev)
    yd = torch.from_numpy(y).to(dev)
    mean = torch.empty(D, dtype=torch.float64, device=dev)
    std = torch.empty(D, dtype=torch.float64, device=dev)
    _lib.check(lib.rs_standardizer_fit(Xd.data_ptr(), len(y), D, mean.data_ptr(), std.data_ptr(), st),
               "rs_standardizer_fit")
    Xs = torch.empty_like(Xd)
    _lib.check(lib.rs_standardize(Xd.data_ptr(), len(y), D, mean.data_ptr(), std.data_ptr(), Xs.data_ptr(), st),
               "rs_standardize")

    rng = np.random.default_rng(cfg.seed + 1)
    params = init_params(D, cfg.hidden, rng)
    scorer = RankingModelScorer(params, cfg.hidden, mean.cpu().numpy(), std.cpu().numpy(), dev)
    m = torch.zeros_like(scorer.flat)
    v = torch.zeros_like(scorer.flat)
    b1, b2 = float(cfg.betas[0]), float(cfg.betas[1])

    def eval_tau() -> float:
        g = scorer.raw_outputs_features(Xed)
        return kendall_tau_b(-g, ye).tau

    step = 0
    window_lo = 0
    checkpoints = []
    loss_buf = []
    for _epoch in range(cfg.epochs):
        order = rng.permutation(len(y))
        for start in range(0, len(order), cfg.batch_size):
            batch = order[start:start + cfg.batch_size]
            if len(batch) < 2:
                continue
            bt = torch.from_numpy(np.ascontiguousarray(batch, dtype=np.int64)).to(dev, non_blocking=True)
            lo = torch.empty(1, dtype=torch.float64, device=dev)
            step += 1
            _lib.check(lib.rs_linear_train_step(Xs.data_ptr(), bt.data_ptr(), yd.data_ptr(), len(batch), D, cfg.hidden,
                                                cfg.bucket_width, scorer.flat.data_ptr(), m.data_ptr(), v.data_ptr(),
                                                cfg.learning_rate, b1, b2, 1e-8, step, lo.data_ptr(), None, st),
                       "rs_linear_train_step")
            loss_buf.append(lo)
            if step % cfg.checkpoint_every == 0:
                window = torch.cat(loss_buf[window_lo:]).cpu().tolist()
                checkpoints.append({"step": step, "train_loss": sum(window) / len(window), "eval_tau": eval_tau()})
                window_lo = len(loss_buf)
    report = {"kind": "ranking", "steps": step, "checkpoints": checkpoints, "eval_tau": eval_tau(),
              "n_train": len(y), "n_eval": len(ye)}
    return TrainResult(scorer, report)
