"""Optimizers with the reference `tpcost.nn` API (nn.py:127-167).

`Adam(names, ...).step(params, grads, lr)` keeps the reference contract:
params / grads are dicts of float64 numpy arrays and params are updated in
place.  The update runs on the GPU in float64 (`tpcb_optimizer_step_f64`,
optim.cu) with the reference's exact operation sequence, so the caller's
parameters and the m / v moments follow the reference trajectory bit for
bit.  The training loops (`costmodel.train/finetune`) instead keep fp32
parameters, m and v resident on the device and never round-trip.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib, engine


class _FlatState:
    """Flat float64 layout of the parameter dict, fixed at the first step;
    every later step checks that the names and shapes are unchanged (the
    reference's per-name m / v would fail the same way on a changed dict)."""

    def __init__(self, names, params):
        self.names = list(names)
        self.shapes = {n: np.shape(params[n]) for n in self.names}
        self.sizes = {n: int(np.prod(self.shapes[n])) for n in self.names}
        self.n = sum(self.sizes.values())

    def check(self, params) -> None:
        if list(params.keys()) != self.names:
            unknown = [n for n in params if n not in self.shapes]
            if unknown:
                raise KeyError(unknown[0])
            raise ValueError("parameter set changed between optimizer steps")
        for n in self.names:
            if np.shape(params[n]) != self.shapes[n]:
                raise ValueError(f"shape of '{n}' changed between optimizer steps")

    def flat(self, tensors) -> np.ndarray:
        if not self.names:
            return np.zeros(0)
        return np.concatenate([np.asarray(tensors[n], dtype=np.float64).ravel()
                               for n in self.names])

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

    def _opt(self):
        raise NotImplementedError

    def _bias_corrections(self):
        return 1.0, 1.0

    def step(self, params: dict, grads: dict, lr: float) -> None:
        engine._need_cuda()
        self.t += 1
        if self._state is None:
            # the reference steps every entry of `params` (nn.py:144) and keys
            # m / v by the names it was built with
            for n in params:
                if n not in self.param_names:
                    raise KeyError(n)
            self._state = _FlatState(list(params.keys()), params)
            n = self._state.n
            self._m = torch.zeros(n, dtype=torch.float64, device="cuda")
            self._v = torch.zeros(n, dtype=torch.float64, device="cuda")
        st = self._state
        st.check(params)
        missing = [n for n in st.names if n not in grads]
        if missing:
            raise KeyError(missing[0])
        p = torch.from_numpy(st.flat(params)).cuda()
        g = torch.from_numpy(st.flat(grads)).cuda()
        bc1, bc2 = self._bias_corrections()
        _lib.check(_lib.load().tpcb_optimizer_step_f64(
            st.n, p.data_ptr(), g.data_ptr(), self._m.data_ptr(), self._v.data_ptr(),
            C.byref(self._opt()), float(lr), bc1, bc2, engine.stream_ptr()), "optimizer_f64")
        st.scatter(p.cpu().numpy(), params)


class Adam(_DeviceOptimizer):
    def __init__(self, param_names, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 weight_decay: float = 0.0):
        super().__init__(param_names, weight_decay)
        self.beta1, self.beta2, self.eps = beta1, beta2, eps

    def _opt(self):
        return engine.optim_struct("adam", self.beta1, self.beta2, self.eps, self.weight_decay)

    def _bias_corrections(self):
        return 1.0 - self.beta1 ** self.t, 1.0 - self.beta2 ** self.t


class Sgd(_DeviceOptimizer):
    def _opt(self):
        return engine.optim_struct("sgd", weight_decay=self.weight_decay)
