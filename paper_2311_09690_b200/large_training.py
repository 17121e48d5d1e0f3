"""Training through the large-model path (csrc/large.cu) — the trainer
`training.train` uses when the fused one-CTA-per-sample kernels cannot hold
the model (full_reference_config: d 716, 11 layers, 46.7 M parameters).

Same semantics as the fused Trainer (costmodel.py:669-780): the reference's
per-bucket minibatch plan (plan_epoch, data-parallel shares when a
communicator is given) and, for fine-tuning, the same-leaf-count target
draws; hybrid / mse / mape loss in the transformed or original space; the
CMD term over [zs; zt] (alpha_cmd > 0 with a target set, single GPU);
Adam / SGD on the flat fp32 parameters, per-epoch validation MAPE / RMSE.
Per step: tpcb_large_loss_backward (source + target forward, loss, CMD,
backward of both passes, every GEMM a 3xTF32 tcgen05 GEMM) → NCCL
all-reduce of the gradient (world > 1) → tpcb_optimizer_step →
tpcb_large_prepare (rebuild the weight image)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib, engine
from .errors import UnsupportedConfig


def large_order(n_leaf: np.ndarray, idx: np.ndarray, with_pos: bool = False):
    """batch indices in bucket order (stable by leaf count) + token offsets
    (+ the input position of each bucket-order row)"""
    idx = np.asarray(idx, dtype=np.int64)
    L = np.asarray(n_leaf, dtype=np.int64)[idx]
    o = np.argsort(L, kind="stable")
    tok = np.zeros(len(idx) + 1, dtype=np.int32)
    np.cumsum(L[o], out=tok[1:])
    out = np.ascontiguousarray(idx[o], dtype=np.int32), tok
    return out + (np.ascontiguousarray(o, dtype=np.int32),) if with_pos else out


class LargeTrainer:
    """Mirrors training.Trainer's interface (plan / run_epoch / evaluate_async
    / collect / tensors) for run_loop."""

    def __init__(self, config, tensors: dict, train_rag: engine.RaggedHost, targets: np.ndarray,
                 loss_struct, valid_rag: engine.RaggedHost | None = None,
                 valid_latency: np.ndarray | None = None, normalizer=None, device="cuda",
                 comm: "engine.Comm | None" = None,
                 target_rag: engine.RaggedHost | None = None):
        from .costmodel import device_model
        use_cmd = target_rag is not None and loss_struct.alpha_cmd > 0
        if use_cmd and comm is not None and comm.world > 1:
            raise UnsupportedConfig("CMD fine-tuning on the large path runs on one GPU")
        self.lib = _lib.load()
        self.config = config
        self.dm = device_model(config)
        self.dev = torch.device(device)
        self.P = self.dm.upload(tensors, device)
        self.m = torch.zeros_like(self.P)
        self.v = torch.zeros_like(self.P)
        self.grad = torch.zeros_like(self.P)
        self.status = engine.Status(self.dev)
        self.src = engine.DeviceSamples(train_rag, config.n_leaf_max, self.status, y=targets,
                                        device=device)
        self.n_leaf = np.asarray(train_rag.n_leaf)
        self.loss = loss_struct
        self.opt = engine.optim_struct(config.optimizer, weight_decay=config.weight_decay)
        self.comm = comm
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.use_cmd = use_cmd
        self.tgt = None
        if use_cmd:
            self.tgt = engine.DeviceSamples(target_rag, config.n_leaf_max, self.status,
                                            device=device)
            self.tgt_leaf = np.asarray(target_rag.n_leaf)
            buckets = {}
            for i, L in enumerate(self.tgt_leaf.tolist()):
                buckets.setdefault(L, []).append(i)
            self.tgt_buckets = {k: np.asarray(v) for k, v in buckets.items()}
        self.stream = torch.cuda.current_stream(self.dev)
        # weight image (forward + backward operands), zero-filled once
        self.path = engine.LargePath(self.dm, self.P, with_backward=True)
        bs = config.batch_size
        l_cap = int(self.n_leaf.max())
        ws = C.c_size_t()
        lt = int(self.tgt_leaf.max()) if use_cmd else 0
        _lib.check(self.lib.tpcb_large_train_ws(self.dm.handle, bs, bs * l_cap,
                                                bs if use_cmd else 0, bs * lt, C.byref(ws)),
                   "large_train_ws")
        self.ws = torch.empty(ws.value, dtype=torch.uint8, device=self.dev)
        self.loss_dev = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.cmd_dev = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.t = 0
        self.valid = valid_rag
        self.valid_lat = None if valid_latency is None else np.asarray(valid_latency, np.float64)
        self.normalizer = normalizer
        self.losses = None
        self._met = None

    def plan(self, rng: np.random.Generator):
        from .training import plan_epoch
        return plan_epoch(rng, self.n_leaf, self.config.batch_size, self.world, self.rank,
                          self.tgt_buckets if self.use_cmd else None,
                          len(self.tgt_leaf) if self.use_cmd else 0)

    def step(self, idx: np.ndarray, n_norm: int, lr: float, d_plan=None,
             tidx: np.ndarray | None = None) -> None:
        """one optimizer step on this rank's share `idx` of a global batch
        (d_plan: device copies (order, tok_off) already on the stream;
        tidx: the step's CMD target samples)"""
        order, tok, pos = large_order(self.n_leaf, idx, with_pos=True)
        s = engine.stream_ptr()
        d_idx, d_tok = (None, None) if d_plan is None else d_plan
        tb = None
        if self.use_cmd and tidx is not None and len(tidx):
            t_order, t_tok, t_pos = large_order(self.tgt_leaf, tidx, with_pos=True)
            self._tkeep = (t_order, t_tok, t_pos)
            tb = _lib.LargeBatch()
            tb.x, tb.ast_row = self.tgt.pk.x.data_ptr(), self.tgt.pk.ast_row.data_ptr()
            tb.devfeat = self.tgt.devfeat.data_ptr()
            tb.h_idx = t_order.ctypes.data_as(C.c_void_p)
            tb.h_tok_off = t_tok.ctypes.data_as(C.c_void_p)
            tb.h_pos = t_pos.ctypes.data_as(C.c_void_p)
            tb.n = len(t_order)
        if len(order):
            _lib.check(self.lib.tpcb_large_loss_backward(
                self.dm.handle, self.P.data_ptr(), self.path.image.data_ptr(),
                self.src.pk.x.data_ptr(), self.src.pk.ast_row.data_ptr(),
                self.src.devfeat.data_ptr(), self.src.y.data_ptr(),
                order.ctypes.data_as(C.c_void_p), tok.ctypes.data_as(C.c_void_p), d_idx, d_tok,
                len(order), C.byref(self.loss), float(n_norm),
                pos.ctypes.data_as(C.c_void_p), C.byref(tb) if tb is not None else None,
                self.ws.data_ptr(), self.ws.numel(), self.grad.data_ptr(),
                self.loss_dev.data_ptr(), self.cmd_dev.data_ptr() if tb is not None else None,
                self.status.ptr, s),
                "large_loss_backward")

        else:
            self.grad.zero_()
            self.loss_dev.zero_()
        if self.comm is not None and self.world > 1:
            _lib.check(self.lib.tpcb_nccl_allreduce_sum(self.comm.handle, self.grad.data_ptr(),
                                                        self.grad.numel(), 0, s), "allreduce")
        self.t += 1
        _lib.check(self.lib.tpcb_optimizer_step(self.dm.handle, self.dm.n_params,
                                                self.P.data_ptr(), None, self.grad.data_ptr(),
                                                self.m.data_ptr(), self.v.data_ptr(),
                                                C.byref(self.opt), float(lr), self.t, s),
                   "optimizer_step")
        self.path.prepare()

    def run_epoch(self, lr: float, flat: np.ndarray, steps: np.ndarray, profile=None) -> int:
        n = steps.shape[0]
        self.losses = torch.zeros(max(n, 1), dtype=torch.float64, device=self.dev)
        self.cmds = torch.zeros(max(n, 1), dtype=torch.float64, device=self.dev)
        # the whole epoch's bucket orders / token offsets in one pinned upload
        # (per-step pageable copies would synchronise the stream every step)
        plans, parts, off = [], [], 0
        for k in range(n):
            o, ns = int(steps[k, 0]), int(steps[k, 1])
            order, tok = large_order(self.n_leaf, flat[o:o + ns])
            plans.append((off, off + len(order)))
            parts += [order, tok]
            off += len(order) + len(tok)
        host = torch.from_numpy(np.concatenate(parts).astype(np.int32) if parts
                                else np.zeros(1, np.int32)).pin_memory()
        dev = host.to(self.dev, non_blocking=True)
        self._epoch_plan = (host, dev)  # keep alive until the epoch's work is done
        for k in range(n):
            o, ns, nt, n_norm = (int(v) for v in steps[k, :4])
            a, b = plans[k]
            self.step(flat[o:o + ns], n_norm, lr,
                      d_plan=(dev[a:].data_ptr(), dev[b:].data_ptr()),
                      tidx=flat[o + ns:o + ns + nt] if self.use_cmd else None)
            self.losses[k:k + 1].copy_(self.loss_dev)
            if self.use_cmd:
                self.cmds[k:k + 1].copy_(self.cmd_dev)
        return n

    def evaluate_async(self) -> None:
        self._met = None
        if self.valid is None or self.normalizer is None:
            return
        rows, ordering, leaf_off, devfeat = engine.upload_ragged(self.valid, self.dev)
        pk = engine.pack(rows, ordering, leaf_off, self.valid.n_ast, self.config.n_leaf_max,
                         self.valid.encoded, self.status)
        _, _, _, _, lat = self.path.forward(pk, self.valid.n_leaf, devfeat, self.status,
                                            self.normalizer, latents=False)
        self._met = lat

    def collect(self, n_steps: int, epoch: int):
        self.status.check("train", epoch)
        losses = self.losses[:n_steps].cpu().numpy() if n_steps else np.zeros(0)
        if not np.all(np.isfinite(losses)):
            from .errors import NonFiniteLoss
            raise NonFiniteLoss(epoch)
        met = np.array([np.inf, np.inf, 0.0])
        if self._met is not None:
            pred = self._met.cpu().numpy()
            y = self.valid_lat
            rel = (pred - y) / y
            met = np.array([float(np.mean(np.abs(rel))), float(np.sqrt(np.mean((pred - y) ** 2))),
                            0.0])
        cmds = self.cmds[:n_steps].cpu().numpy() if (self.use_cmd and n_steps) else \
            np.zeros(n_steps)
        return losses, cmds, met

    def tensors(self, flat: torch.Tensor | None = None) -> dict:
        return self.dm.unflatten((self.P if flat is None else flat).double().cpu().numpy())


def large_loss_backward(params, rag: engine.RaggedHost, y: np.ndarray, idx=None,
                        mode: str = "hybrid", lambda_hybrid: float = 1e-3, offset: float = 0.0,
                        n_norm: int | None = None, mape_space: str = "transformed",
                        normalizer=None, alpha_cmd: float = 0.0, cmd_order: int = 5,
                        target_rag: engine.RaggedHost | None = None):
    """One batch's (loss, gradient dict, CMD value) through the large path —
    the costmodel.backward drop-in for large configs (costmodel.py:529-570;
    no optimizer step).  With alpha_cmd > 0 and a target set the CMD term
    couples the two forward passes."""
    from .costmodel import device_model
    lib = _lib.load()
    cfg = params.config
    dm = device_model(cfg)
    P = dm.upload(params.tensors)
    status = engine.Status(P.device)
    src = engine.DeviceSamples(rag, cfg.n_leaf_max, status, y=np.asarray(y, np.float64))
    path = engine.LargePath(dm, P, with_backward=True)
    idx = np.arange(rag.n_ast) if idx is None else np.asarray(idx)
    order, tok, pos = large_order(rag.n_leaf, idx, with_pos=True)
    use_cmd = alpha_cmd > 0 and target_rag is not None
    tb, n_t, tok_t = None, 0, 0
    if use_cmd:
        tgt = engine.DeviceSamples(target_rag, cfg.n_leaf_max, status)
        t_order, t_tok, t_pos = large_order(target_rag.n_leaf, np.arange(target_rag.n_ast),
                                            with_pos=True)
        tb = _lib.LargeBatch()
        tb.x, tb.ast_row, tb.devfeat = tgt.pk.x.data_ptr(), tgt.pk.ast_row.data_ptr(), \
            tgt.devfeat.data_ptr()
        tb.h_idx = t_order.ctypes.data_as(C.c_void_p)
        tb.h_tok_off = t_tok.ctypes.data_as(C.c_void_p)
        tb.h_pos = t_pos.ctypes.data_as(C.c_void_p)
        tb.n = n_t = len(t_order)
        tok_t = int(t_tok[-1])
    ws = C.c_size_t()
    _lib.check(lib.tpcb_large_train_ws(dm.handle, len(order), int(tok[-1]), n_t, tok_t,
                                       C.byref(ws)), "large_train_ws")
    wsb = torch.empty(ws.value, dtype=torch.uint8, device=P.device)
    grad = torch.empty_like(P)
    loss_dev = torch.zeros(1, dtype=torch.float64, device=P.device)
    cmd_dev = torch.zeros(1, dtype=torch.float64, device=P.device)
    loss = engine.loss_struct(mode, lambda_hybrid, offset, alpha_cmd if use_cmd else 0.0,
                              cmd_order, mape_space, normalizer)
    _lib.check(lib.tpcb_large_loss_backward(
        dm.handle, P.data_ptr(), path.image.data_ptr(), src.pk.x.data_ptr(),
        src.pk.ast_row.data_ptr(), src.devfeat.data_ptr(), src.y.data_ptr(),
        order.ctypes.data_as(C.c_void_p), tok.ctypes.data_as(C.c_void_p), None, None,
        len(order), C.byref(loss), float(n_norm or len(order)), pos.ctypes.data_as(C.c_void_p),
        C.byref(tb) if tb is not None else None, wsb.data_ptr(), wsb.numel(), grad.data_ptr(),
        loss_dev.data_ptr(), cmd_dev.data_ptr(), status.ptr, engine.stream_ptr()),
        "large_loss_backward")
    status.check("large_loss_backward")
    return (float(loss_dev.item()), dm.unflatten(grad.double().cpu().numpy()),
            float(cmd_dev.item()))
