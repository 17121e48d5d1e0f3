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


# ---------------------------------------------------------------------------
# persistence: the reference's JSONL (dataset.py:421-485) and a binary ragged
# SoA that loads straight into a CompactBatch
# ---------------------------------------------------------------------------

def _fmt(x: float) -> str:
    if not math.isfinite(x):
        raise ValidationError("cannot serialize non-finite float")
    return format(float(x), ".17g")


def sample_to_line(s: Sample) -> str:
    """One JSONL record, byte-identical to the reference's (dataset.py:427-448)."""
    import json
    c = s.compact
    vectors = "[" + ",".join("[" + ",".join(_fmt(v) for v in row) + "]"
                             for row in np.asarray(c.leaf_vectors)) + "]"
    return ("{" f"\"id\":{json.dumps(s.id)},\"task_id\":{json.dumps(s.task_id)},"
            f"\"model_id\":{json.dumps(s.model_id)},\"device_id\":{json.dumps(s.device_id)},"
            f"\"n_leaf\":{c.n_leaf},\"vectors\":{vectors},"
            f"\"ordering\":[{','.join(str(int(i)) for i in c.ordering)}],"
            f"\"serialized\":[{','.join(str(int(i)) for i in c.serialized)}],"
            f"\"latency_s\":{_fmt(s.latency_s)}" "}")


def save_dataset(ds: Dataset, path) -> None:
    with open(path, "w", encoding="utf-8") as f:
        for s in ds.samples:
            f.write(sample_to_line(s))
            f.write("\n")


def load_dataset(path) -> Dataset:
    """Reference JSONL reader (dataset.py:451-485), same validation."""
    import json
    from .features import CompactAst
    samples = []
    with open(path, "r", encoding="utf-8") as f:
        for lineno, line in enumerate(f, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                d = json.loads(line)
            except json.JSONDecodeError as e:
                raise ValidationError(f"{path}:{lineno}: bad JSON: {e}") from e
            vec = np.asarray(d["vectors"], dtype=np.float64)
            if vec.ndim != 2:
                raise ValidationError("vectors must be a 2-D array")
            c = CompactAst(leaf_vectors=vec, ordering=tuple(int(i) for i in d["ordering"]),
                           serialized=tuple(int(i) for i in d["serialized"]),
                           n_leaf=int(d["n_leaf"]))
            if c.n_leaf != vec.shape[0]:
                raise ValidationError("n_leaf does not match vector count")
            samples.append(Sample(id=str(d["id"]), task_id=str(d["task_id"]),
                                  model_id=str(d["model_id"]), device_id=str(d["device_id"]),
                                  compact=c, latency_s=float(d["latency_s"])))
    return Dataset(samples=samples)


_SPLIT_CODE = {None: 0, "train": 1, "valid": 2, "test": 3, "holdout": 4}
_SPLIT_NAME = {v: k for k, v in _SPLIT_CODE.items()}


def save_dataset_bin(ds: Dataset, path) -> None:
    """Ragged SoA .npz: vectors (T,24) f64, ordering (T,) i32, serialized
    (S,) i32, n_leaf / n_ser (B,), latency_s (B,) f64, string ids, split codes.
    Bit-exact round trip of everything the JSONL holds (and the splits)."""
    cs = [s.compact for s in ds.samples]
    np.savez(path,
             vectors=(np.concatenate([np.asarray(c.leaf_vectors, np.float64) for c in cs])
                      if cs else np.zeros((0, 24))),
             ordering=np.array([i for c in cs for i in c.ordering], dtype=np.int32),
             serialized=np.array([i for c in cs for i in c.serialized], dtype=np.int32),
             n_leaf=np.array([c.n_leaf for c in cs], dtype=np.int64),
             n_ser=np.array([len(c.serialized) for c in cs], dtype=np.int64),
             latency_s=np.array([s.latency_s for s in ds.samples], dtype=np.float64),
             id=np.array([s.id for s in ds.samples], dtype=np.str_),
             task_id=np.array([s.task_id for s in ds.samples], dtype=np.str_),
             model_id=np.array([s.model_id for s in ds.samples], dtype=np.str_),
             device_id=np.array([s.device_id for s in ds.samples], dtype=np.str_),
             split=np.array([_SPLIT_CODE[ds.splits.get(s.id)] for s in ds.samples],
                            dtype=np.int8))


def load_batch_bin(path, devices: dict):
    """The binary file straight into the GPU path's input: (CompactBatch,
    latency_s, split codes, ids) with no per-sample Python objects."""
    from .features import CompactBatch
    with np.load(path, allow_pickle=False) as z:
        names = sorted(devices)
        dev_ix = {n: i for i, n in enumerate(names)}
        try:
            di = np.array([dev_ix[d] for d in z["device_id"]], dtype=np.int32)
        except KeyError as e:
            raise ValidationError(f"unknown device {e.args[0]!r}") from None
        batch = CompactBatch(z["vectors"], z["ordering"], z["n_leaf"], di,
                             [devices[n] for n in names])
        return batch, z["latency_s"], z["split"], z["id"]


def load_dataset_bin(path) -> Dataset:
    from .features import CompactAst
    with np.load(path, allow_pickle=False) as z:
        vec, order, ser = z["vectors"], z["ordering"], z["serialized"]
        lo = np.concatenate([[0], np.cumsum(z["n_leaf"])])
        so = np.concatenate([[0], np.cumsum(z["n_ser"])])
        samples, splits = [], {}
        for i in range(z["n_leaf"].shape[0]):
            c = CompactAst(leaf_vectors=vec[lo[i]:lo[i + 1]].copy(),
                           ordering=tuple(int(v) for v in order[lo[i]:lo[i + 1]]),
                           serialized=tuple(int(v) for v in ser[so[i]:so[i + 1]]),
                           n_leaf=int(z["n_leaf"][i]))
            s = Sample(id=str(z["id"][i]), task_id=str(z["task_id"][i]),
                       model_id=str(z["model_id"][i]), device_id=str(z["device_id"][i]),
                       compact=c, latency_s=float(z["latency_s"][i]))
            samples.append(s)
            code = int(z["split"][i])
            if code:
                splits[s.id] = _SPLIT_NAME[code]
    return Dataset(samples=samples, splits=splits)
