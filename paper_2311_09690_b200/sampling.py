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
        if self.kappa < 2:
            return
        # the common case — the running total stays > 0, so every step draws
        # rng.random() — runs with the uniforms pre-drawn and no per-step host
        # synchronisation; a step that saw total == 0 (the reference then
        # draws rng.integers) is replayed exactly from there
        saved = rng.bit_generator.state
        us = np.ascontiguousarray(rng.random(self.kappa - 1))
        zero = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device=self.dev)
        _lib.check(self.lib.tpcb_kmeanspp_steps(self.x.data_ptr(), self.n, self.d, 1, self.kappa,
                                                us.ctypes.data_as(C.c_void_p),
                                                self.centers.data_ptr(), self.closest.data_ptr(),
                                                self.total.data_ptr(), zero.data_ptr(),
                                                self.ws.ptr, self.ws.size, self.s()),
                   "kmeanspp_steps")
        z = int(zero.item())
        if z >= self.kappa:
            return
        rng.bit_generator.state = saved
        rng.random(z - 1)  # the draws of steps 1 .. z-1, as consumed above
        # rebuild the state after step z-1 (the speculative steps ≥ z
        # overwrote closest / total) by re-running steps 1 .. z-1, then step
        # by step with the reference's branch per step
        _lib.check(self.lib.tpcb_kmeanspp_init(self.x.data_ptr(), self.n, self.d, first,
                                               self.centers.data_ptr(), self.closest.data_ptr(),
                                               self.total.data_ptr(), self.ws.ptr, self.ws.size,
                                               self.s()), "kmeanspp_init")
        if z > 1:
            _lib.check(self.lib.tpcb_kmeanspp_steps(self.x.data_ptr(), self.n, self.d, 1, z,
                                                    us.ctypes.data_as(C.c_void_p),
                                                    self.centers.data_ptr(),
                                                    self.closest.data_ptr(),
                                                    self.total.data_ptr(), zero.data_ptr(),
                                                    self.ws.ptr, self.ws.size, self.s()),
                       "kmeanspp_steps")
        for i in range(z, self.kappa):
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


def select_tasks(x, kappa: int, tasks: list, seed: int = 0, init_centers=None,
                 assign: str = "exact") -> list:
    """κ task ids: clusters by size desc (stable), each takes the closest
    remaining task, ties to the earlier task (sampling.py:126-144).
    assign: the clustering's assignment mode (see DeviceKMeans)."""
    if len(tasks) < kappa:
        raise TooFewTasks(f"{len(tasks)} tasks < kappa={kappa}")
    clusters = kmeans(x, kappa, seed=seed, init_centers=init_centers, assign=assign)
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


# ---------------------------------------------------------------------------
# Data-parallel KMeans (SURVEY 8(e), C4 multi-GPU): the points are sharded
# across ranks (rank r holds a contiguous slice of the global point order),
# the centres are replicated.  Per k-means++ centre: one gather of the local
# closest-distance totals, one of the local CDF sums, one of the local search
# hits and a broadcast of the chosen point; per Lloyd iteration: an
# all-reduce of the int32 counts and of the changed flag and one all-gather
# of the [kappa, d] member sums, added in rank order on every rank (so the
# centres are bit-identical on all ranks and independent of the NCCL
# algorithm).  At world size 1 every value is bit-identical to kmeans().
# ---------------------------------------------------------------------------


class _CudaShard:
    """One rank's shard on its GPU: the local pieces between the collectives
    (tpcb_kmeanspp_closest / _cdf / _search, tpcb_kmeans_assign[_tc] /
    _changed / _partial)."""

    def __init__(self, x: np.ndarray, kappa: int, device, assign: str):
        self.km = DeviceKMeans(x, kappa, device, assign)
        self.lib, self.n, self.d, self.kappa = self.km.lib, self.km.n, self.km.d, kappa
        self.x_host, self.device = x, self.km.dev
        self.local_sum = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.found = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.sums = torch.zeros((kappa, self.d), dtype=torch.float64, device=self.device)

    @property
    def assign(self):
        return self.km.assign

    @property
    def assign_prev(self):
        return self.km.assign_prev

    @property
    def counts(self):
        return self.km.counts

    @property
    def own(self):
        return self.km.own

    def closest(self, center: torch.Tensor, init: bool) -> torch.Tensor:
        k = self.km
        _lib.check(self.lib.tpcb_kmeanspp_closest(k.x.data_ptr(), self.n, self.d,
                                                  center.data_ptr(), int(init),
                                                  k.closest.data_ptr(), k.total.data_ptr(),
                                                  k.ws.ptr, k.ws.size, k.s()), "kmeanspp_closest")
        return k.total

    def cdf(self, total: torch.Tensor) -> torch.Tensor:
        k = self.km
        _lib.check(self.lib.tpcb_kmeanspp_cdf(k.closest.data_ptr(), self.n, total.data_ptr(),
                                              self.local_sum.data_ptr(), k.ws.ptr, k.ws.size,
                                              k.s()), "kmeanspp_cdf")
        return self.local_sum

    def search(self, offset: float, total: float, u: float) -> int:
        k = self.km
        _lib.check(self.lib.tpcb_kmeanspp_search(self.n, offset, total, u, self.found.data_ptr(),
                                                 k.ws.ptr, k.ws.size, k.s()), "kmeanspp_search")
        return int(self.found.item())

    def point(self, j: int) -> torch.Tensor:
        return self.km.x[j].clone()

    def assign_step(self, centers: torch.Tensor) -> None:
        self.km.centers.copy_(centers)
        self.km.assign_step()

    def changed(self) -> torch.Tensor:
        k = self.km
        _lib.check(self.lib.tpcb_kmeans_changed(k.assign.data_ptr(), k.assign_prev.data_ptr(),
                                                self.n, k.flag.data_ptr(), k.s()), "kmeans_changed")
        return k.flag

    def save_prev(self) -> None:
        self.km.assign_prev.copy_(self.km.assign)

    def partial(self) -> torch.Tensor:
        k = self.km
        _lib.check(self.lib.tpcb_kmeans_partial(k.x.data_ptr(), self.n, self.d, self.kappa,
                                                k.assign.data_ptr(), k.counts.data_ptr(),
                                                self.sums.data_ptr(), k.ws.ptr, k.ws.size, k.s()),
                   "kmeans_partial")
        return self.sums

    def set_assignment(self, a: np.ndarray, own: np.ndarray) -> None:
        self.km.assign.copy_(torch.from_numpy(a))
        self.km.own.copy_(torch.from_numpy(own))
        self.km.counts.copy_(torch.from_numpy(np.bincount(a, minlength=self.kappa)
                                              .astype(np.int32)))


class ShardedKMeans:
    """k-means++ and Lloyd over point shards with torch.distributed
    collectives (NCCL for CUDA shards).  Every rank draws the same RNG
    sequence (same seed), so the sequential choices of sampling.py:45-60 and
    the empty-cluster repair of sampling.py:90-97 are replayed identically on
    every rank over the concatenated point order."""

    def __init__(self, shard, group=None):
        import torch.distributed as dist
        self.dist, self.group, self.shard = dist, group, shard
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.kappa, self.d, self.dev = shard.kappa, shard.d, shard.device
        ns = self._gather(torch.tensor([shard.n], dtype=torch.int64, device=self.dev))
        self.ns = [int(v) for v in ns]
        if min(self.ns) < 1:
            raise ValidationError("every rank needs at least one point")
        self.start = [sum(self.ns[:r]) for r in range(self.world)]
        self.n_global = sum(self.ns)
        if self.n_global < self.kappa:
            raise TooFewPoints(f"{self.n_global} points < kappa={self.kappa}")
        self.centers = torch.zeros((self.kappa, self.d), dtype=torch.float64, device=self.dev)

    # -- collectives -------------------------------------------------------
    def _gather(self, t: torch.Tensor) -> list:
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return [o.cpu() for o in out] if t.numel() == 1 else out

    def _ordered_sum(self, parts: list) -> torch.Tensor:
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        return acc

    def _bcast_point(self, owner: int, j: int) -> torch.Tensor:
        buf = (self.shard.point(j) if owner == self.rank
               else torch.empty(self.d, dtype=torch.float64, device=self.dev))
        src = owner if self.group is None else self.dist.get_global_rank(self.group, owner)
        self.dist.broadcast(buf, src=src, group=self.group)
        return buf

    def _global_point(self, g: int) -> torch.Tensor:
        owner = max(r for r in range(self.world) if self.start[r] <= g)
        return self._bcast_point(owner, g - self.start[owner])

    # -- k-means++ (sampling.py:45-60) -------------------------------------
    def kmeanspp(self, rng: np.random.Generator) -> None:
        c = self._global_point(int(rng.integers(0, self.n_global)))
        self.centers[0] = c
        total = self._ordered_sum(self._gather(self.shard.closest(self.centers[0], True)))
        for i in range(1, self.kappa):
            if float(total) == 0.0:
                c = self._global_point(int(rng.integers(0, self.n_global)))
            else:
                u = float(rng.random())
                sums = [float(s) for s in self._gather(self.shard.cdf(total.to(self.dev)))]
                offset, tot_p = 0.0, sums[0]
                for r in range(1, self.world):
                    tot_p += sums[r]
                for r in range(self.rank):
                    offset = sums[r] if r == 0 else offset + sums[r]
                j = self.shard.search(offset, tot_p, u)
                found = [int(v) for v in self._gather(
                    torch.tensor([j], dtype=torch.int64, device=self.dev))]
                hits = [r for r in range(self.world) if found[r] >= 0]
                # no hit (u at the rounding edge of the last CDF value): the
                # last point, as the single-device search does
                owner = hits[0] if hits else self.world - 1
                c = self._bcast_point(owner, found[owner] if hits else self.ns[-1] - 1)
            self.centers[i] = c
            total = self._ordered_sum(self._gather(self.shard.closest(self.centers[i], False)))

    # -- Lloyd (sampling.py:63-106) ----------------------------------------
    def _counts_global(self) -> torch.Tensor:
        g = self.shard.counts.clone()
        self.dist.all_reduce(g, group=self.group)  # int32: exact in any order
        return g

    def repair_empty(self, counts: np.ndarray) -> None:
        """Sequential steal of the globally farthest point from a cluster
        with > 1 members (first point in global order on ties)."""
        sh = self.shard
        a = sh.assign.cpu().numpy()
        own = sh.own.cpu().numpy()
        centers = self.centers.cpu().numpy()
        counts = counts.astype(np.int64).copy()
        for c in range(self.kappa):
            if counts[c] != 0:
                continue
            cand = np.flatnonzero(counts[a] > 1)
            if cand.size:
                j = int(cand[own[cand].argmax()])
                mine = torch.tensor([1.0, own[j], float(j), float(a[j])], dtype=torch.float64)
            else:
                mine = torch.tensor([0.0, 0.0, 0.0, 0.0], dtype=torch.float64)
            rows = [r.cpu().numpy() for r in
                    self._gather_rows(mine.to(self.dev))]
            best = -1
            for r in range(self.world):  # strict >: the lowest rank wins ties
                if rows[r][0] > 0 and (best < 0 or rows[r][1] > rows[best][1]):
                    best = r
            j, old = int(rows[best][2]), int(rows[best][3])
            if best == self.rank:
                a[j] = c
                own[j] = _point_dist(sh.x_host[j], centers[c])
            counts[c] += 1
            counts[old] -= 1
        sh.set_assignment(a, own)

    def _gather_rows(self, t: torch.Tensor) -> list:
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return out

    def lloyd(self, max_iter: int = KMEANS_MAX_ITER) -> int:
        it = 0
        for it in range(1, max_iter + 1):
            self.shard.assign_step(self.centers)
            counts = self._counts_global()
            if int(counts.min().item()) == 0:
                self.repair_empty(counts.cpu().numpy())
                counts = self._counts_global()
            flag = self.shard.changed().clone()
            self.dist.all_reduce(flag, op=self.dist.ReduceOp.MAX, group=self.group)
            if not int(flag.item()):
                break
            self.shard.save_prev()
            sums = self._ordered_sum(self._gather_rows(self.shard.partial()))
            live = counts > 0
            self.centers[live] = sums[live] / counts[live].to(torch.float64)[:, None]
        return it


def kmeans_sharded(x_local, kappa: int, seed: int = 0, init_centers=None, assign: str = "exact",
                   group=None, shard=None) -> ClusterModel:
    """kmeans() over the points of all ranks (this rank holds `x_local`, a
    contiguous slice of the global point order, in rank order).  Returns the
    replicated centres, THIS rank's assignment and the global sizes.
    `shard` overrides the local backend (default: this rank's GPU)."""
    x_local = np.asarray(x_local, dtype=np.float64)
    if x_local.ndim == 1:
        x_local = x_local[:, None]
    if kappa < 1:
        raise ValidationError("kappa must be >= 1")
    if shard is None:
        shard = _CudaShard(np.ascontiguousarray(x_local), kappa,
                           torch.device("cuda", torch.cuda.current_device()), assign)
    km = ShardedKMeans(shard, group)
    if init_centers is not None:
        centers = np.asarray(init_centers, dtype=np.float64).copy()
        if centers.ndim == 1:
            centers = centers[:, None]
        if centers.shape != (kappa, x_local.shape[1]):
            raise DimensionMismatch("init_centers shape mismatch")
        km.centers.copy_(torch.from_numpy(centers))
    else:
        km.kmeanspp(np.random.default_rng(seed))
    km.lloyd()
    a = shard.assign_prev.cpu().numpy()
    if np.any(a < 0):
        a = shard.assign.cpu().numpy()
    sizes = torch.from_numpy(np.bincount(a, minlength=kappa).astype(np.int64)).to(shard.device)
    km.dist.all_reduce(sizes, group=group)
    return ClusterModel(centers=km.centers.cpu().numpy(), assignment=a, sizes=sizes.cpu().numpy())
