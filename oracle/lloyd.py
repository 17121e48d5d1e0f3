"""Oracle: k-means task sampler, float64, chunked (test infrastructure).

Restates sampling.py:40-144 with identical floating-point semantics but
without the (n, κ, d) temporary of `_pairwise_dist` (which needs 268 GB at
1M × 1024 × 32), so it also serves as the chunked CPU restatement for
configs the reference itself cannot run.

  distance       sqrt of numpy's pairwise sum of (x-c)² over d   sampling.py:40-42
  k-means++      rng.integers then rng.choice(n, p=closest/total)  sampling.py:45-60
  Lloyd          argmin (first index), empty-cluster steal, stop when the
                 assignment is unchanged (tested before the update), ≤300 it.
                                                                   sampling.py:63-106
  Ψ table        mean over a task's rows of the distance          sampling.py:109-123
  select_tasks   clusters by size desc (stable), min (Ψ, task)    sampling.py:126-144
"""

from __future__ import annotations

import numpy as np

MAX_ITER = 300  # sampling.py:13


def distances(x: np.ndarray, centers: np.ndarray, chunk: int = 4096) -> np.ndarray:
    """Full (n, κ) distance matrix, chunked over rows."""
    out = np.empty((x.shape[0], centers.shape[0]))
    for a in range(0, x.shape[0], chunk):
        diff = x[a:a + chunk, None, :] - centers[None, :, :]
        out[a:a + chunk] = np.sqrt((diff ** 2).sum(axis=2))
    return out


def assign(x: np.ndarray, centers: np.ndarray, chunk: int = 4096):
    """(argmin index, own distance) per point, never materialising (n, κ)."""
    n = x.shape[0]
    idx = np.empty(n, dtype=np.int64)
    own = np.empty(n)
    for a in range(0, n, chunk):
        diff = x[a:a + chunk, None, :] - centers[None, :, :]
        dist = np.sqrt((diff ** 2).sum(axis=2))
        j = dist.argmin(axis=1)
        idx[a:a + chunk] = j
        own[a:a + chunk] = dist[np.arange(j.size), j]
    return idx, own


def point_dist(xi: np.ndarray, c: np.ndarray) -> float:
    diff = xi[None, None, :] - c[None, None, :]
    return float(np.sqrt((diff ** 2).sum(axis=2))[0, 0])


def kmeanspp(x: np.ndarray, kappa: int, rng: np.random.Generator) -> np.ndarray:
    """k-means++ seeding with the reference's exact RNG consumption."""
    n = x.shape[0]
    centers = np.empty((kappa, x.shape[1]))
    centers[0] = x[int(rng.integers(0, n))]
    closest = ((x - centers[0]) ** 2).sum(axis=1)
    for i in range(1, kappa):
        tot = closest.sum()
        if tot == 0.0:
            j = int(rng.integers(0, n))
        else:
            cdf = np.cumsum(closest / tot)
            cdf /= cdf[-1]
            j = int(cdf.searchsorted(rng.random(), side="right"))
        centers[i] = x[j]
        closest = np.minimum(closest, ((x - centers[i]) ** 2).sum(axis=1))
    return centers


def repair_empty(x, centers, a, own, kappa):
    """Sequential empty-cluster repair (sampling.py:90-97)."""
    for c in range(kappa):
        counts = np.bincount(a, minlength=kappa)
        if counts[c] == 0:
            cand = np.flatnonzero(counts[a] > 1)
            steal = cand[own[cand].argmax()]
            a[steal] = c
            own[steal] = point_dist(x[steal], centers[c])
    return a, own


def member_means(x, a, kappa, centers):
    """centers[c] = mean of members in index order (sequential row sum / m)."""
    order = np.argsort(a, kind="stable")
    counts = np.bincount(a, minlength=kappa)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    xs = x[order]
    for c in range(kappa):
        m = counts[c]
        if m:
            acc = xs[starts[c]].copy()
            for r in range(1, m):
                acc += xs[starts[c] + r]
            centers[c] = acc / m
    return centers


def kmeans(x, kappa: int, seed: int = 0, init_centers=None):
    """Returns (centers, assignment, sizes, n_iter)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    n = x.shape[0]
    rng = np.random.default_rng(seed)
    if init_centers is not None:
        centers = np.asarray(init_centers, dtype=np.float64).copy()
        if centers.ndim == 1:
            centers = centers[:, None]
    else:
        centers = kmeanspp(x, kappa, rng)
    assignment = np.full(n, -1, dtype=np.int64)
    it = 0
    for it in range(1, MAX_ITER + 1):
        a, own = assign(x, centers)
        a, own = repair_empty(x, centers, a, own, kappa)
        if np.array_equal(a, assignment):
            break
        assignment = a
        centers = member_means(x, assignment, kappa, centers)
    sizes = np.bincount(assignment, minlength=kappa)
    return centers, assignment, sizes, it


def psi_table(centers: np.ndarray, task_feats: list[np.ndarray]) -> np.ndarray:
    psi = np.empty((centers.shape[0], len(task_feats)))
    for t, f in enumerate(task_feats):
        d = distances(np.asarray(f, dtype=np.float64), centers)
        acc = d[0].copy()
        for r in range(1, d.shape[0]):
            acc += d[r]
        psi[:, t] = acc / d.shape[0]
    return psi


def greedy_pick(psi: np.ndarray, sizes: np.ndarray) -> list[int]:
    order = np.argsort(-sizes, kind="stable")
    left = list(range(psi.shape[1]))
    picked = []
    for e in order:
        best = min(left, key=lambda t: (psi[e, t], t))
        picked.append(best)
        left.remove(best)
    return picked
