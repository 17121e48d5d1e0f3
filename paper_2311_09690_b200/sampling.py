"""KMeans task sampler on the GPU — the reference `tpcost.sampling` API
(sampling.py:16-144).

kmeans: k-means++ seeding (host draws the reference's exact RNG sequence,
device evaluates closest distances / totals / the CDF search), then Lloyd
iterations (device assignment + member means, host only for the sequential
empty-cluster repair of sampling.py:90-97, which the reference also runs
point by point).  build_distance_table: device Ψ.  select_tasks: clusters
by size, greedy min (Ψ, task) — host (κ sequential picks).
All arithmetic is float64 with the reference's summation order, so results
are bit-identical (see csrc/kmeans.cu).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, engine
from .errors import DimensionMismatch, TooFewPoints, TooFewTasks, ValidationError

KMEANS_MAX_ITER = 300


@dataclass
class ClusterModel:
    centers: np.ndarray
    assignment: np.ndarray
    sizes: np.ndarray


@dataclass
class TaskFeatureSet:
    task_id: str
    features: np.ndarray

    def validate(self) -> None:
        if self.features.ndim != 2 or self.features.shape[0] == 0:
            raise ValidationError(f"task '{self.task_id}' needs a non-empty 2-D feature array")


@dataclass
class DistanceTable:
    psi: np.ndarray
    task_ids: list


class _Ws:
    def __init__(self, n, d, kappa, device):
        sz = C.c_size_t()
        _lib.check(_lib.load().tpcb_kmeans_ws_size(n, d, kappa, C.byref(sz)), "kmeans_ws")
        self.buf = torch.empty(sz.value, dtype=torch.uint8, device=device)

    @property
    def ptr(self):
        return self.buf.data_ptr()

    @property
    def size(self):
        return self.buf.numel()


def _point_dist(xi: np.ndarray, c: np.ndarray) -> float:
    """One distance by the reference formula (for the host repair path)."""
    diff = xi[None, None, :] - c[None, None, :]
    return float(np.sqrt((diff ** 2).sum(axis=2))[0, 0])


class DeviceKMeans:
    """x resident on the device; k-means++ and Lloyd steps as kernel calls."""

    def __init__(self, x: np.ndarray, kappa: int, device="cuda", assign: str = "exact"):
        """assign: "exact" (float64, bit-identical to the reference) or "tc"
        (3xTF32 tensor-core distance GEMM + exact float64 re-rank of the top-4
        candidates; d <= 32; >= 99.9 % agreement, see tpcb_kmeans_assign_tc)."""
        engine._need_cuda()
        if assign not in ("exact", "tc"):
            raise ValidationError(f"unknown assign mode {assign!r}")
        self.lib = _lib.load()
        self.x_host = x
        self.n, self.d = x.shape
        self.kappa = kappa
        self.dev = torch.device(device)
        self.x = torch.from_numpy(np.ascontiguousarray(x)).to(self.dev)
        self.centers = torch.zeros((kappa, self.d), dtype=torch.float64, device=self.dev)
        self.closest = torch.empty(self.n, dtype=torch.float64, device=self.dev)
        self.total = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.assign = torch.full((self.n,), -1, dtype=torch.int64, device=self.dev)
        self.assign_prev = torch.full((self.n,), -1, dtype=torch.int64, device=self.dev)
        self.own = torch.empty(self.n, dtype=torch.float64, device=self.dev)
        self.counts = torch.zeros(kappa, dtype=torch.int32, device=self.dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.ws = _Ws(self.n, self.d, kappa, self.dev)
        self.assign_mode = assign if self.d <= 32 else "exact"
        if self.assign_mode == "tc":
            nb = int(self.lib.tpcb_kmeans_assign_tc_ws(kappa))
            self.tc_ws = torch.empty(nb, dtype=torch.uint8, device=self.dev)

    def s(self):
        return engine.stream_ptr()

    def kmeanspp(self, rng: np.random.Generator) -> None:
        """sampling._kmeans_pp_init with the same RNG calls."""
        first = int(rng.integers(0, self.n))
        _lib.check(self.lib.tpcb_kmeanspp_init(self.x.data_ptr(), self.n, self.d, first,
                                               self.centers.data_ptr(), self.closest.data_ptr(),
                                               self.total.data_ptr(), self.ws.ptr, self.ws.size,
                                               self.s()), "kmeanspp_init")
        for i in range(1, self.kappa):
            total = float(self.total.item())
            if total == 0.0:
                u, direct = -1.0, int(rng.integers(0, self.n))
            else:
                u, direct = float(rng.random()), -1
            _lib.check(self.lib.tpcb_kmeanspp_step(self.x.data_ptr(), self.n, self.d, i, u, direct,
                                                   self.centers.data_ptr(),
                                                   self.closest.data_ptr(), self.total.data_ptr(),
                                                   None, self.ws.ptr, self.ws.size, self.s()),
                       "kmeanspp_step")

    def assign_step(self) -> None:
        if self.assign_mode == "tc":
            _lib.check(self.lib.tpcb_kmeans_assign_tc(
                self.x.data_ptr(), self.n, self.d, self.centers.data_ptr(), self.kappa,
                self.assign.data_ptr(), self.own.data_ptr(), self.counts.data_ptr(),
                self.tc_ws.data_ptr(), self.tc_ws.numel(), self.s()), "kmeans_assign_tc")
            return
        _lib.check(self.lib.tpcb_kmeans_assign(self.x.data_ptr(), self.n, self.d,
                                               self.centers.data_ptr(), self.kappa,
                                               self.assign.data_ptr(), self.own.data_ptr(),
                                               self.counts.data_ptr(), self.s()), "kmeans_assign")

    def repair_empty(self) -> None:
        """Sequential empty-cluster repair (sampling.py:90-97), host side —
        only reached when some cluster received no point."""
        a = self.assign.cpu().numpy()
        own = self.own.cpu().numpy()
        centers = self.centers.cpu().numpy()
        for c in range(self.kappa):
            counts = np.bincount(a, minlength=self.kappa)
            if counts[c] == 0:
                cand = np.flatnonzero(counts[a] > 1)
                steal = cand[own[cand].argmax()]
                a[steal] = c
                own[steal] = _point_dist(self.x_host[steal], centers[c])
        self.assign.copy_(torch.from_numpy(a))
        self.own.copy_(torch.from_numpy(own))
        self.counts.copy_(torch.from_numpy(np.bincount(a, minlength=self.kappa).astype(np.int32)))

    def changed(self) -> bool:
        _lib.check(self.lib.tpcb_kmeans_changed(self.assign.data_ptr(), self.assign_prev.data_ptr(),
                                                self.n, self.flag.data_ptr(), self.s()),
                   "kmeans_changed")
        return bool(self.flag.item())

    def update(self) -> None:
        _lib.check(self.lib.tpcb_kmeans_update(self.x.data_ptr(), self.n, self.d, self.kappa,
                                               self.assign.data_ptr(), self.counts.data_ptr(),
                                               self.centers.data_ptr(), self.ws.ptr, self.ws.size,
                                               self.s()), "kmeans_update")

    def lloyd(self, max_iter: int = KMEANS_MAX_ITER) -> int:
        it = 0
        for it in range(1, max_iter + 1):
            self.assign_step()
            if int(self.counts.min().item()) == 0:
                self.repair_empty()
            if not self.changed():
                break
            self.assign_prev.copy_(self.assign)
            self.update()
        # the converged assignment equals assign_prev (unchanged) or, after
        # max_iter, the last accepted one
        return it


def kmeans(x, kappa: int, seed: int = 0, init_centers=None, assign: str = "exact") -> ClusterModel:
    """Lloyd's iterations from a k-means++ start (sampling.py:63-106).
    assign="tc": tensor-core assignment mode (see DeviceKMeans)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    n = x.shape[0]
    if kappa < 1:
        raise ValidationError("kappa must be >= 1")
    if n < kappa:
        raise TooFewPoints(f"{n} points < kappa={kappa}")
    rng = np.random.default_rng(seed)
    km = DeviceKMeans(x, kappa, assign=assign)
    if init_centers is not None:
        centers = np.asarray(init_centers, dtype=np.float64).copy()
        if centers.ndim == 1:
            centers = centers[:, None]
        if centers.shape != (kappa, x.shape[1]):
            raise DimensionMismatch("init_centers shape mismatch")
        km.centers.copy_(torch.from_numpy(centers))
    else:
        km.kmeanspp(rng)
    km.lloyd()
    assignment = km.assign_prev.cpu().numpy()
    if np.any(assignment < 0):  # converged on the very first pass cannot happen;
        assignment = km.assign.cpu().numpy()  # max_iter == 0 guard
    sizes = np.bincount(assignment, minlength=kappa)
    return ClusterModel(centers=km.centers.cpu().numpy(), assignment=assignment, sizes=sizes)


def build_distance_table(clusters: ClusterModel, tasks: list) -> DistanceTable:
    """Ψ[e, t] = mean L2 distance of task t's features to centre e (device)."""
    if not tasks:
        raise TooFewTasks("need at least one task")
    d = clusters.centers.shape[1]
    feats = []
    for task in tasks:
        task.validate()
        f = np.asarray(task.features, dtype=np.float64)
        if f.shape[1] != d:
            raise DimensionMismatch(f"task '{task.task_id}' has dim {f.shape[1]}, centers {d}")
        feats.append(f)
    engine._need_cuda()
    off = np.zeros(len(feats) + 1, dtype=np.int64)
    np.cumsum([f.shape[0] for f in feats], out=off[1:])
    fd = torch.from_numpy(np.ascontiguousarray(np.concatenate(feats))).cuda()
    od = torch.from_numpy(off).cuda()
    cd = torch.from_numpy(np.ascontiguousarray(clusters.centers, dtype=np.float64)).cuda()
    kappa = clusters.centers.shape[0]
    psi = torch.empty((kappa, len(feats)), dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().tpcb_distance_table(fd.data_ptr(), od.data_ptr(), len(feats), d,
                                               cd.data_ptr(), kappa, psi.data_ptr(),
                                               engine.stream_ptr()), "distance_table")
    return DistanceTable(psi=psi.cpu().numpy(), task_ids=[t.task_id for t in tasks])


def select_tasks(x, kappa: int, tasks: list, seed: int = 0, init_centers=None) -> list:
    """κ task ids: clusters by size desc (stable), each takes the closest
    remaining task, ties to the earlier task (sampling.py:126-144)."""
    if len(tasks) < kappa:
        raise TooFewTasks(f"{len(tasks)} tasks < kappa={kappa}")
    clusters = kmeans(x, kappa, seed=seed, init_centers=init_centers)
    table = build_distance_table(clusters, tasks)
    order = np.argsort(-clusters.sizes, kind="stable")
    taken = np.zeros(len(tasks), dtype=bool)
    selected = []
    for e in order:
        row = np.where(taken, np.inf, table.psi[e])
        best = int(np.argmin(row))  # first index among equal minima
        selected.append(table.task_ids[best])
        taken[best] = True
    return selected
