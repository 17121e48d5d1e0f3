"""Optimizers with the reference `tpcost.nn` API (nn.py:127-167), stepping a
flat fp32 parameter vector on the GPU (optim.cu).

`Adam(names, ...).step(params, grads, lr)` keeps the reference contract —
params/grads are dicts of numpy arrays and params are updated in place — for
drop-in use; the training loops (`costmodel.train/finetune`) instead keep
parameters, m and v resident on the device and never round-trip.
"""

from __future__ import annotations

import numpy as np
import torch

from . import engine


class _FlatState:
    def __init__(self, names, params):
        self.names = list(names)
        self.shapes = {n: np.asarray(params[n]).shape for n in self.names}
        self.sizes = {n: int(np.prod(self.shapes[n])) for n in self.names}
        self.n = sum(self.sizes.values())

    def flat(self, tensors) -> np.ndarray:
        return np.concatenate([np.asarray(tensors[n], dtype=np.float64).ravel()
                               for n in self.names]) if self.names else np.zeros(0)

    def scatter(self, flat, params) -> None:
        o = 0
        for n in self.names:
            k = self.sizes[n]
            params[n][...] = flat[o:o + k].reshape(self.shapes[n])
            o += k


class _DeviceOptimizer:
    kind: str = ""

    def __init__(self, param_names, weight_decay: float = 0.0):
        self.param_names = list(param_names)
        self.weight_decay = weight_decay
        self.t = 0
        self._state = None
        self._m = self._v = None
        self._dm = None

    def _opt(self):
        raise NotImplementedError

    def step(self, params: dict, grads: dict, lr: float) -> None:
        engine._need_cuda()
        self.t += 1
        names = [n for n in self.param_names if n in params]
        if self._state is None:
            self._state = _FlatState(names, params)
            n = self._state.n
            self._m = torch.zeros(n, dtype=torch.float32, device="cuda")
            self._v = torch.zeros(n, dtype=torch.float32, device="cuda")
            self._dm = None  # bare flat vector: no model handle needed
        st = self._state
        p = torch.from_numpy(st.flat(params).astype(np.float32)).cuda()
        g = torch.from_numpy(st.flat(grads).astype(np.float32)).cuda()
        engine.optimizer_step(self._dm, p, None, g, self._m, self._v, self._opt(), lr, self.t)
        st.scatter(p.double().cpu().numpy(), params)


class Adam(_DeviceOptimizer):
    def __init__(self, param_names, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 weight_decay: float = 0.0):
        super().__init__(param_names, weight_decay)
        self.beta1, self.beta2, self.eps = beta1, beta2, eps

    def _opt(self):
        return engine.optim_struct("adam", self.beta1, self.beta2, self.eps, self.weight_decay)


class Sgd(_DeviceOptimizer):
    def _opt(self):
        return engine.optim_struct("sgd", weight_decay=self.weight_decay)
