"""Oracle: the reference training step, float64 (test infrastructure / the
CPU-baseline arm of bench.py).

One step = costmodel.backward on a single-bucket batch (costmodel.py:529-570)
followed by nn.Adam.step over every tensor (nn.py:136-154), exactly the
reference `train` inner loop body (costmodel.py:700-706).  Used to time the
reference algorithm on the GPU box's host cores (the reference package itself
is not shipped to the box) and to cross-check the device trainer.
"""

from __future__ import annotations

import numpy as np

from . import predictor as op


class AdamState:
    def __init__(self, T: dict, b1=0.9, b2=0.999, eps=1e-8, wd=0.0):
        self.m = {k: np.zeros_like(v) for k, v in T.items()}
        self.v = {k: np.zeros_like(v) for k, v in T.items()}
        self.t = 0
        self.b1, self.b2, self.eps, self.wd = b1, b2, eps, wd

    def step(self, T: dict, G: dict, lr: float) -> None:
        self.t += 1
        bc1 = 1.0 - self.b1 ** self.t
        bc2 = 1.0 - self.b2 ** self.t
        for k, p in T.items():
            g = G.get(k)
            if g is None:
                g = np.zeros_like(p)
            if self.wd:
                g = g + self.wd * p
            m, v = self.m[k], self.v[k]
            m *= self.b1
            m += (1.0 - self.b1) * g
            v *= self.b2
            v += (1.0 - self.b2) * g * g
            p -= lr * (m / bc1) / (np.sqrt(v / bc2) + self.eps)


def train_step(T: dict, dm: op.Dims, x: np.ndarray, dev: np.ndarray, y: np.ndarray,
               opt: AdamState, lr: float, offset: float, lam: float = 1e-3) -> float:
    """x: (n, L, 24) encoded rows of one bucket, dev (n, 6), y (n,) model space."""
    pred, _, _, _, tape = op.bucket_forward(T, dm, x, dev)
    value, dpred = op.loss_and_grad(pred, y, "hybrid", lam, offset)
    G: dict = {}
    op.bucket_backward(T, dm, tape, dpred, None, G)
    opt.step(T, G, lr)
    return value
