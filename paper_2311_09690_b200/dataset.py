"""Label normalisation and the dataset containers `train()` consumes.

Mirrors the parts of `tpcost.dataset` the predictor path touches:
`BoxCoxNormalizer` (dataset.py:69-115; its bulk decode is fused into the
forward kernel, this class is the host-side parameter holder), `fit_boxcox`
(dataset.py:145-169, host-side, once per training run), `Sample` /
`Dataset` / `split_dataset` (dataset.py:42-61, 181-213).  The synthetic
program generator lives in `synth.py` (vectorised, for benchmarks).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy import stats as sstats

from .errors import DegenerateLabels, DomainError, EmptyDataset, NotFitted, ValidationError

_LAMBDA_ZERO_EPS = 1e-9


@dataclass
class Sample:
    id: str
    task_id: str
    model_id: str
    device_id: str
    compact: object
    latency_s: float


@dataclass
class Dataset:
    samples: list = field(default_factory=list)
    splits: dict = field(default_factory=dict)

    def subset(self, split: str) -> list:
        return [s for s in self.samples if self.splits.get(s.id) == split]

    def labels(self, split: str | None = None) -> np.ndarray:
        samples = self.samples if split is None else self.subset(split)
        return np.array([s.latency_s for s in samples], dtype=np.float64)


@dataclass
class BoxCoxNormalizer:
    """((y+shift)^λ − 1)/λ (log at λ≈0), then standardised (dataset.py:69-115)."""

    lambda_bc: float = 0.0
    shift: float = 0.0
    fitted: bool = False
    t_mean: float = 0.0
    t_std: float = 1.0
    loss_offset: float = 0.0

    def _check(self) -> None:
        if not self.fitted:
            raise NotFitted("normalizer used before fit")

    def transform(self, y):
        self._check()
        arr = np.asarray(y, dtype=np.float64) + self.shift
        if np.any(arr <= 0):
            raise DomainError("transform input must be > -shift")
        if abs(self.lambda_bc) < _LAMBDA_ZERO_EPS:
            out = np.log(arr)
        else:
            out = (np.power(arr, self.lambda_bc) - 1.0) / self.lambda_bc
        return float(out) if np.isscalar(y) else out

    def inverse_transform(self, t):
        self._check()
        arr = np.asarray(t, dtype=np.float64)
        if abs(self.lambda_bc) < _LAMBDA_ZERO_EPS:
            out = np.exp(arr) - self.shift
        else:
            base = self.lambda_bc * arr + 1.0
            if np.any(base <= 0):
                raise DomainError("no positive preimage: lambda*t + 1 <= 0")
            out = np.power(base, 1.0 / self.lambda_bc) - self.shift
        return float(out) if np.isscalar(t) else out

    def encode(self, y):
        return (self.transform(y) - self.t_mean) / self.t_std

    def decode(self, e):
        return self.inverse_transform(np.asarray(e) * self.t_std + self.t_mean)


def _golden_max(f, lo: float, hi: float, tol: float) -> float:
    g = (math.sqrt(5.0) - 1.0) / 2.0
    a, b = lo, hi
    c, d = b - g * (b - a), a + g * (b - a)
    fc, fd = f(c), f(d)
    while b - a > tol:
        if fc > fd:
            b, d, fd = d, c, fc
            c = b - g * (b - a)
            fc = f(c)
        else:
            a, c, fc = c, d, fd
            d = a + g * (b - a)
            fd = f(d)
    return (a + b) / 2.0


def fit_boxcox(train_labels, lambda_range=(-2.0, 2.0), tol: float = 1e-5) -> BoxCoxNormalizer:
    """Profile-likelihood Box-Cox fit by golden-section search, then
    standardisation (dataset.py:145-169)."""
    y = np.asarray(train_labels, dtype=np.float64)
    if y.size < 2 or np.unique(y).size < 2:
        raise DegenerateLabels("need at least 2 distinct labels")
    if np.any(y < 0):
        raise ValidationError("labels must be positive")
    shift = 1e-12 if np.any(y == 0) else 0.0
    lam = _golden_max(lambda l: float(sstats.boxcox_llf(l, y + shift)), lambda_range[0],
                      lambda_range[1], tol)
    norm = BoxCoxNormalizer(lambda_bc=lam, shift=shift, fitted=True)
    t = norm.transform(y)
    t_std = float(np.std(t))
    if t_std == 0.0:
        raise DegenerateLabels("transformed labels are constant")
    norm.t_mean = float(np.mean(t))
    norm.t_std = t_std
    norm.loss_offset = 1.0 - float(np.min((t - norm.t_mean) / t_std))
    return norm


def split_dataset(ds: Dataset, ratios=(8, 1, 1), seed: int = 0,
                  holdout_models=frozenset()) -> Dataset:
    """Seeded train/valid/test assignment (dataset.py:181-213)."""
    if not ds.samples:
        raise EmptyDataset("cannot split an empty dataset")
    if min(ratios) < 0 or sum(ratios) <= 0:
        raise ValidationError("ratios must be non-negative with positive sum")
    splits: dict = {}
    rest = []
    for s in ds.samples:
        if s.model_id in holdout_models:
            splits[s.id] = "holdout"
        else:
            rest.append(s)
    order = np.random.default_rng(seed).permutation(len(rest))
    total = sum(ratios)
    n = len(rest)
    n_valid = round(n * ratios[1] / total)
    n_test = round(n * ratios[2] / total)
    n_train = n - n_valid - n_test
    for pos, idx in enumerate(order):
        splits[rest[idx].id] = ("train" if pos < n_train else
                                "valid" if pos < n_train + n_valid else "test")
    return Dataset(samples=ds.samples, splits=splits)
