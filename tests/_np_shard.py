"""Test-only CPU shard backend for sampling.ShardedKMeans: the same local
pieces as the CUDA shard (_CudaShard), in numpy with the oracle's
arithmetic, on CPU tensors so the gloo backend can run the collectives.
This exercises the host orchestration (collective sequence, offsets, owner
choice, ordered sums, distributed empty-cluster repair) without a GPU."""

import numpy as np
import torch

from oracle import lloyd


class NumpyShard:
    def __init__(self, x: np.ndarray, kappa: int):
        self.x_host = np.ascontiguousarray(x, dtype=np.float64)
        self.n, self.d = self.x_host.shape
        self.kappa = kappa
        self.device = torch.device("cpu")
        self.closest_v = np.zeros(self.n)
        self.cdf_v = np.zeros(self.n)
        self.assign = torch.full((self.n,), -1, dtype=torch.int64)
        self.assign_prev = torch.full((self.n,), -1, dtype=torch.int64)
        self.own = torch.zeros(self.n, dtype=torch.float64)
        self.counts = torch.zeros(kappa, dtype=torch.int32)

    def closest(self, center, init):
        dsq = ((self.x_host - center.numpy()) ** 2).sum(axis=1)
        self.closest_v = dsq if init else np.minimum(self.closest_v, dsq)
        return torch.tensor([self.closest_v.sum()], dtype=torch.float64)

    def cdf(self, total):
        self.cdf_v = np.cumsum(self.closest_v / float(total))
        return torch.tensor([self.cdf_v[-1]], dtype=torch.float64)

    def search(self, offset, total, u):
        hit = np.flatnonzero((offset + self.cdf_v) / total > u)
        return int(hit[0]) if hit.size else -1

    def point(self, j):
        return torch.from_numpy(self.x_host[j].copy())

    def assign_step(self, centers):
        a, own = lloyd.assign(self.x_host, centers.numpy())
        self.set_assignment(a, own)

    def set_assignment(self, a, own):
        self.assign = torch.from_numpy(np.asarray(a, dtype=np.int64).copy())
        self.own = torch.from_numpy(np.asarray(own, dtype=np.float64).copy())
        self.counts = torch.from_numpy(np.bincount(a, minlength=self.kappa).astype(np.int32))

    def changed(self):
        return torch.tensor([int(not torch.equal(self.assign, self.assign_prev))],
                            dtype=torch.int32)

    def save_prev(self):
        self.assign_prev = self.assign.clone()

    def partial(self):
        a = self.assign.numpy()
        sums = np.zeros((self.kappa, self.d))
        order = np.argsort(a, kind="stable")
        for c in range(self.kappa):
            mem = order[a[order] == c]
            if mem.size:
                acc = self.x_host[mem[0]].copy()
                for r in mem[1:]:
                    acc += self.x_host[r]
                sums[c] = acc
        return torch.from_numpy(sums)
