"""Oracle: Adam / SGD steps over a flat parameter vector (test infra).

Restates nn.py:127-167: L2 weight decay added to the gradient, β=(0.9,
0.999), eps 1e-8, bias-corrected step, every tensor updated every step
(zero gradients still decay m/v), plus the cyclic learning-rate triangle of
costmodel.py:617-623.
"""

from __future__ import annotations

import numpy as np


def adam_step(p, g, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8, wd=0.0):
    """In-place on p, m, v (1-D float64); t is the 1-based step count."""
    if wd:
        g = g + wd * p
    m *= b1
    m += (1.0 - b1) * g
    v *= b2
    v += (1.0 - b2) * g * g
    bc1 = 1.0 - b1 ** t
    bc2 = 1.0 - b2 ** t
    p -= lr * (m / bc1) / (np.sqrt(v / bc2) + eps)


def sgd_step(p, g, lr, wd=0.0):
    if wd:
        g = g + wd * p
    p -= lr * g


def lr_at(lr, schedule, epoch):
    if schedule == "constant":
        return lr
    floor = lr / 10.0
    return floor + (lr - floor) * (1.0 - abs((epoch % 20) / 10.0 - 1.0))
