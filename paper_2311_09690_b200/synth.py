"""Vectorised synthetic compact-AST generator for benchmarks.

Same generative model as the reference's `generate_synthetic`
(dataset.py:245-414) — tasks of 32 programs sharing a template (1..6 leaf
chains of 1..3 loops under a root loop, per-leaf op/byte counts, annotation
probabilities 0.15/0.25/0.15 and 0.4 parallel at the root, per-leaf log2
iteration target e_center ± 1.5 split across the chain with extents clamped
to 1..512), compact-AST vectors per the 24-entry schema of
features.compute_vector (features.py:168-203), serialized-position ordering
of the marker pre-order walk (features.py:206-245) and roofline latency
labels (dataset.py:245-270) — but drawn with array operations, so 1M ASTs take
seconds instead of minutes.  The RNG stream differs from the reference's, so
samples are distributionally equivalent, not identical; parity tests use the
reference's own golden samples (tests/golden), never this generator.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MAX_LEAVES = 6
MAX_CHAIN = 3
MAX_BITS = 9.0


@dataclass
class SynthSet:
    vectors: np.ndarray   # (n_tok, 24) float64
    ordering: np.ndarray  # (n_tok,) int32
    n_leaf: np.ndarray    # (n,) int64
    latency: np.ndarray   # (n,) float64 seconds
    task: np.ndarray      # (n,) int64

    @property
    def n(self) -> int:
        return int(self.n_leaf.shape[0])

    def offsets(self) -> np.ndarray:
        off = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(self.n_leaf, out=off[1:])
        return off

    def take(self, idx) -> "SynthSet":
        idx = np.asarray(idx, dtype=np.int64)
        off = self.offsets()
        lens = self.n_leaf[idx]
        starts = off[idx]
        rows = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + \
            np.arange(int(lens.sum()))
        return SynthSet(self.vectors[rows], self.ordering[rows], self.n_leaf[idx],
                        self.latency[idx], self.task[idx])


def _annot(rng, shape, p_par):
    return (rng.random(shape) < p_par, rng.random(shape) < 0.25, rng.random(shape) < 0.15)


def _log_count(rng, shape, bits):
    return np.round(2.0 ** rng.uniform(0.0, bits, size=shape))


def generate(n: int, seed: int = 0, task_size: int = 32, peak_gflops: float = 2048.0,
             bandwidth_gbps: float = 1024.0, cores: int = 16, flops_eff: float = 0.6,
             mem_eff: float = 0.7, per_leaf_overhead: float = 2e-6) -> SynthSet:
    """n synthetic samples on one device (DEFAULT_SYNTH_DEVICE numbers)."""
    rng = np.random.default_rng(seed)
    n_tasks = (n + task_size - 1) // task_size
    T, Lm, Cm = n_tasks, MAX_LEAVES, MAX_CHAIN
    # ---------------------------------------------------------- templates
    t_nleaf = rng.integers(1, MAX_LEAVES + 1, size=T)
    t_chain = rng.integers(1, MAX_CHAIN + 1, size=(T, Lm))
    c_par, c_vec, c_unr = _annot(rng, (T, Lm, Cm), 0.15)
    r_par, r_vec, r_unr = _annot(rng, T, 0.4)
    fma = _log_count(rng, (T, Lm), 9.0)
    add = _log_count(rng, (T, Lm), 5.0)
    mul = _log_count(rng, (T, Lm), 5.0)
    div = rng.integers(0, 3, size=(T, Lm)).astype(np.float64)
    spc = rng.integers(0, 3, size=(T, Lm)).astype(np.float64)
    brd = 4.0 * _log_count(rng, (T, Lm), 5.0)
    bwr = 4.0 * _log_count(rng, (T, Lm), 3.0)
    nbr = rng.integers(1, 5, size=(T, Lm)).astype(np.float64)
    nbw = rng.integers(1, 3, size=(T, Lm)).astype(np.float64)
    e_center = rng.uniform(10.0, 20.0, size=T)
    # ---------------------------------------------------------- instances
    task = np.repeat(np.arange(T), task_size)[:n]
    N = n
    nleaf = t_nleaf[task]
    chain = t_chain[task]                       # (N, Lm)
    e_root = rng.uniform(2.0, 6.0, size=N)
    e_target = e_center[task][:, None] + rng.uniform(-1.5, 1.5, size=(N, Lm))
    # split (e_target - e_root) bits over the chain, each in [0, 9]
    remaining = np.minimum(e_target - e_root[:, None], MAX_BITS * chain)
    bits = np.zeros((N, Lm, Cm))
    u = rng.random((N, Lm, Cm))
    for i in range(Cm):
        active = i < chain
        left = chain - i - 1
        lo = np.maximum(0.0, remaining - MAX_BITS * left)
        hi = np.minimum(MAX_BITS, remaining)
        e = np.where(hi > lo, lo + (hi - lo) * u[..., i], hi)
        e = np.where(active, e, 0.0)
        bits[..., i] = e
        remaining = remaining - e
    ext = np.clip(np.round(2.0 ** bits), 1, 512)          # (N, Lm, Cm)
    ext = np.where(np.arange(Cm)[None, None, :] < chain[..., None], ext, 1.0)
    root_ext = np.clip(np.round(2.0 ** e_root), 1, 512)   # (N,)
    # ---------------------------------------------------------- vectors
    valid_c = np.arange(Cm)[None, None, :] < chain[..., None]
    prod = root_ext[:, None] * np.prod(ext, axis=2)        # iterations per leaf
    inner = np.take_along_axis(ext, (chain - 1)[..., None], axis=2)[..., 0]
    v = np.zeros((N, Lm, 24))
    v[..., 0] = 1 + chain
    v[..., 1] = np.log2(1 + prod)
    v[..., 2] = np.log2(1 + inner)
    v[..., 3] = np.log2(1 + root_ext)[:, None]
    for k, (cf, rf) in enumerate(((c_vec, r_vec), (c_unr, r_unr), (c_par, r_par))):
        tag = cf[task] & valid_c
        cnt = tag.sum(axis=2) + rf[task][:, None]
        p = np.prod(np.where(tag, ext, 1.0), axis=2) * np.where(rf[task], root_ext, 1.0)[:, None]
        v[..., 4 + k] = cnt
        v[..., 7 + k] = np.where(cnt > 0, np.log2(1 + p), 0.0)
    f, a, m, dv, sp = fma[task], add[task], mul[task], div[task], spc[task]
    for k, c in enumerate((f, a, m, dv, sp)):
        v[..., 10 + k] = np.log2(1 + c)
    per_iter = 2 * f + a + m + dv + sp
    tot_flops = per_iter * prod
    rd, wr = brd[task] * prod, bwr[task] * prod
    v[..., 15] = np.log2(1 + tot_flops)
    v[..., 16] = np.log2(1 + brd[task])
    v[..., 17] = np.log2(1 + bwr[task])
    v[..., 18] = np.log2(1 + rd)
    v[..., 19] = np.log2(1 + wr)
    v[..., 20] = nbr[task]
    v[..., 21] = nbw[task]
    v[..., 22] = tot_flops / (rd + wr + 1)
    v[..., 23] = np.arange(Lm)[None, :] / nleaf[:, None]
    # serialized position of leaf i: root + Σ_{i'<i}(chain+2) + chain_i
    step = chain + 2
    before = np.concatenate([np.zeros((N, 1)), np.cumsum(step, axis=1)[:, :-1]], axis=1)
    order = (1 + before + chain).astype(np.int32)
    # ---------------------------------------------------------- labels
    flops_rate = peak_gflops * 1e9 * flops_eff
    bytes_rate = bandwidth_gbps * 1e9 / 8.0 * mem_eff
    fl = 2.0 ** v[..., 15] - 1.0
    nb = 2.0 ** v[..., 18] - 1.0 + 2.0 ** v[..., 19] - 1.0
    par = np.where(v[..., 6] > 0, np.maximum(np.minimum(float(cores), 2.0 ** v[..., 9] - 1.0), 1.0),
                   1.0)
    leaf_t = np.maximum(fl / (flops_rate * par), nb / bytes_rate)
    leaf_mask = np.arange(Lm)[None, :] < nleaf[:, None]
    lat = per_leaf_overhead * nleaf + np.where(leaf_mask, leaf_t, 0.0).sum(axis=1)
    return SynthSet(vectors=v[leaf_mask], ordering=order[leaf_mask],
                    n_leaf=nleaf.astype(np.int64), latency=lat, task=task.astype(np.int64))


def split(n: int, seed: int = 0, ratios=(8, 1, 1)):
    """Seeded 8:1:1 index split (dataset.split_dataset's rounding)."""
    order = np.random.default_rng(seed).permutation(n)
    tot = sum(ratios)
    n_valid = round(n * ratios[1] / tot)
    n_test = round(n * ratios[2] / tot)
    n_train = n - n_valid - n_test
    return order[:n_train], order[n_train:n_train + n_valid], order[n_train + n_valid:]
