"""Device-resident training loops: `train` and `finetune` of costmodel.py:669-780.

Parameters, transposed weights, Adam moments and both datasets (K1-packed)
live on the GPU for the whole run.  Per epoch the host does only what the
reference does on the host and nothing more:

  * the seeded batch plan (`_epoch_batches`, costmodel.py:632-645) and, for
    fine-tuning, the same-leaf-count target draws (costmodel.py:759-766) —
    identical RNG calls, hence identical batch composition;
  * one upload of that plan, one native call running every step of the epoch
    (tpcb_train_epoch: per step fused fwd/bwd(+CMD) → fixed-order gradient
    reduction + Adam/SGD → transposed-weight refresh), one device-side
    validation pass (fused forward + Box-Cox decode + metrics kernel), and a
    single synchronisation to read the per-step losses and the metrics.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, engine
from .errors import EmptyDataset, NonFiniteLoss, ValidationError


@dataclass
class EpochLog:
    epoch: int
    train_loss: float
    val_mape: float
    val_rmse: float
    lr: float
    cmd: float = 0.0


@dataclass
class TrainResult:
    params: object
    normalizer: object
    log: list
    best_epoch: int
    best_val_mape: float


def lr_at(config, epoch: int) -> float:
    """Constant or triangular cyclic schedule (costmodel.py:617-623)."""
    if config.lr_schedule == "constant":
        return config.lr
    floor = config.lr / 10.0
    tri = 1.0 - abs((epoch % 20) / 10.0 - 1.0)
    return floor + (config.lr - floor) * tri


def epoch_batches(rng: np.random.Generator, n_leaves: np.ndarray, batch_size: int) -> list:
    """Shuffled single-bucket minibatches — same RNG calls, same batches as
    costmodel._epoch_batches (costmodel.py:632-645)."""
    n_leaves = np.asarray(n_leaves)
    order = np.argsort(n_leaves, kind="stable")
    sorted_l = n_leaves[order]
    batches = []
    for L in np.unique(sorted_l):
        idx = order[sorted_l == L]
        idx = idx[rng.permutation(len(idx))]
        for s in range(0, len(idx), batch_size):
            batches.append(idx[s:s + batch_size])
    perm = rng.permutation(len(batches))
    return [batches[i] for i in perm]


def plan_epoch(rng: np.random.Generator, n_leaf: np.ndarray, batch_size: int, world: int = 1,
               rank: int = 0, tgt_buckets: dict | None = None, n_tgt: int = 0,
               dp_mode: str = "weak"):
    """One epoch's batch plan for `rank` of `world` data-parallel ranks.

    Every rank draws the same global plan — `epoch_batches`
    (costmodel.py:632-645) and, for fine-tuning, the same-leaf-count target
    draw per batch (costmodel.py:762-766) — and keeps its contiguous share
    (np.array_split) of each global batch.  dp_mode:
      "strong"  the global batch is the reference's batch_size: each
                reference batch is split across the ranks, so the epoch has
                the reference's optimizer steps and batch composition at any
                world size;
      "weak"    the global batch is batch_size × world (batch_size per rank;
                the reference's semantics at that larger batch size).
    Returns (flat int32 sample indices, int32 [n_steps, 8] step table:
    offset, n_src, n_tgt, n_norm = global batch, src_pos, ns_glob, tgt_pos,
    nt_glob)."""
    if dp_mode not in ("weak", "strong"):
        raise ValidationError(f"unknown data-parallel mode '{dp_mode}'")
    gbs = batch_size * world if dp_mode == "weak" else batch_size
    batches = epoch_batches(rng, n_leaf, gbs)
    parts, steps, off = [], [], 0
    for b in batches:
        tsel = np.zeros(0, dtype=np.int64)
        if tgt_buckets is not None:
            pool = tgt_buckets.get(int(n_leaf[b[0]]))
            if pool is None or len(pool) == 0:
                pool = np.arange(n_tgt)
            take = min(gbs, len(pool))
            picked = rng.choice(len(pool), size=take, replace=False)
            tsel = pool[np.sort(picked)]
        sb = np.array_split(b, world)
        st = np.array_split(tsel, world)
        sp = int(sum(len(c) for c in sb[:rank]))
        tp = int(sum(len(c) for c in st[:rank]))
        parts.append(sb[rank])
        parts.append(st[rank])
        steps.append((off, len(sb[rank]), len(st[rank]), len(b), sp, len(b), tp, len(tsel)))
        off += len(sb[rank]) + len(st[rank])
    flat = np.concatenate(parts).astype(np.int32) if parts else np.zeros(0, np.int32)
    return flat, np.asarray(steps, dtype=np.int32).reshape(-1, 8)


class Trainer:
    """Training state resident on cuda:0 (or the current device)."""

    def __init__(self, config, tensors: dict, train_rag: engine.RaggedHost,
                 targets: np.ndarray, loss_struct, valid_rag: engine.RaggedHost | None = None,
                 valid_latency: np.ndarray | None = None, normalizer=None,
                 target_rag: engine.RaggedHost | None = None, device="cuda",
                 use_graph: bool = True, comm: "engine.Comm | None" = None,
                 overlap: bool = True, dp_mode: str = "weak", wgrad_tc: bool = False):
        from .costmodel import device_model
        self.config = config
        self.dm = device_model(config)
        self.dev = torch.device(device)
        self.P = self.dm.upload(tensors, device)
        self.PT = torch.empty_like(self.P)
        engine.transpose_params(self.dm, self.P, self.PT)
        self.m = torch.zeros_like(self.P)
        self.v = torch.zeros_like(self.P)
        self.status = engine.Status(self.dev)
        n_max = config.n_leaf_max
        self.src = engine.DeviceSamples(train_rag, n_max, self.status, y=targets, device=device)
        self.tgt = None
        self.use_cmd = config.alpha_cmd > 0 and target_rag is not None
        if self.use_cmd:
            self.tgt = engine.DeviceSamples(target_rag, n_max, self.status, device=device)
            self.tgt_leaf = target_rag.n_leaf
            self.tgt_buckets = {}
            for i, L in enumerate(self.tgt_leaf.tolist()):
                self.tgt_buckets.setdefault(L, []).append(i)
            self.tgt_buckets = {k: np.asarray(v) for k, v in self.tgt_buckets.items()}
        self.loss = loss_struct
        self.opt = engine.optim_struct(config.optimizer, weight_decay=config.weight_decay)
        # data parallel: every rank takes a contiguous share of each global
        # batch (plan_epoch dp_mode: "weak" = batch_size per rank, "strong" =
        # the reference's batch split across ranks); gradients reduced every
        # step in rank order (capi_train.cu)
        self.comm = comm
        self.dp_mode = dp_mode
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        rows = config.batch_size * (2 if self.use_cmd else 1)
        l_cap = int(np.max(train_rag.n_leaf))
        if target_rag is not None:
            l_cap = max(l_cap, int(np.max(target_rag.n_leaf)))
        self.ws = engine.TrainWorkspace(self.dm, rows, device, z_rows=rows * self.world,
                                        l_cap=l_cap, overlap=overlap and comm is None,
                                        wgrad_tc=wgrad_tc)
        self.grad = torch.zeros_like(self.P) if comm is not None else None
        self.n_train = train_rag.n_ast
        self.n_leaf = np.asarray(train_rag.n_leaf)
        # plan buffers (fixed sizes: every epoch visits every training sample once)
        n_steps_max = int(sum(-(-int(c) // config.batch_size)
                              for c in np.bincount(self.n_leaf)[1:]))  # ≥ global steps
        self.max_entries = self.n_train + (n_steps_max * config.batch_size if self.use_cmd else 0)
        self.batch_dev = torch.zeros(max(self.max_entries, 1), dtype=torch.int32, device=device)
        self.batch_host = torch.zeros(max(self.max_entries, 1), dtype=torch.int32).pin_memory()
        self.hyper_dev = torch.zeros(2, dtype=torch.float64, device=device)  # lr, t0 (as f64)
        self.t0_dev = torch.zeros(1, dtype=torch.int64, device=device)
        self.t = 0
        self.steps_dev = None
        self.valid = None
        if valid_rag is not None:
            rows_, ordering, leaf_off, devfeat = engine.upload_ragged(valid_rag, device)
            self.valid_pk = engine.pack(rows_, ordering, leaf_off, valid_rag.n_ast, n_max,
                                        valid_rag.encoded, self.status,
                                        int(_lib.load().tpcb_forward_rows(self.dm.handle)))
            self.valid_devfeat = devfeat
            self.valid_y = torch.from_numpy(np.asarray(valid_latency, dtype=np.float64)).to(device)
            self.valid = valid_rag
        self.normalizer = normalizer
        self.metrics_dev = torch.zeros(3, dtype=torch.float64, device=device)
        # a dedicated (capturable) stream; the captured epoch graph replays on it
        self.stream = torch.cuda.Stream(device=self.dev)
        self.stream.wait_stream(torch.cuda.current_stream(self.dev))
        self.graph = None
        if use_graph:
            h = C.c_void_p()
            _lib.check(_lib.load().tpcb_graph_create(C.byref(h)), "graph_create")
            self.graph = h

    def __del__(self):
        try:
            if getattr(self, "graph", None):
                torch.cuda.synchronize()
                _lib.load().tpcb_graph_destroy(self.graph)
                self.graph = None
        except Exception:
            pass

    # ------------------------------------------------------------ planning
    def plan(self, rng: np.random.Generator):
        """Host batch plan of this rank for one epoch (see plan_epoch)."""
        return plan_epoch(rng, self.n_leaf, self.config.batch_size, self.world, self.rank,
                          self.tgt_buckets if self.use_cmd else None,
                          len(self.tgt_leaf) if self.use_cmd else 0, self.dp_mode)

    # ------------------------------------------------------------ one epoch
    def run_epoch(self, lr: float, flat: np.ndarray, steps: np.ndarray, profile=None):
        """Enqueue one epoch.  profile: a float64 numpy array of 3 to run it
        uncaptured with per-kernel-class device timing (ms)."""
        with torch.cuda.stream(self.stream):
            return self._run_epoch(lr, flat, steps, profile)

    def _run_epoch(self, lr: float, flat: np.ndarray, steps: np.ndarray, profile=None):
        n_steps = steps.shape[0]
        if flat.size > self.batch_host.numel():
            raise ValidationError("epoch plan larger than the planned buffer")
        self.batch_host[:flat.size].copy_(torch.from_numpy(flat))
        self.batch_dev[:flat.size].copy_(self.batch_host[:flat.size], non_blocking=True)
        if self.steps_dev is None or self.steps_dev.shape[0] < n_steps:
            self.steps_dev = torch.zeros((max(n_steps, 1), 8), dtype=torch.int32, device=self.dev)
            self.step_loss = torch.zeros(max(n_steps, 1), dtype=torch.float64, device=self.dev)
            self.step_cmd = torch.zeros(max(n_steps, 1), dtype=torch.float64, device=self.dev)
        self.steps_dev[:n_steps].copy_(torch.from_numpy(steps))
        self.hyper_dev[0] = lr
        self.t0_dev[0] = self.t
        plan = _lib.Plan()
        plan.d_batch, plan.d_steps, plan.n_steps = (self.batch_dev.data_ptr(),
                                                    self.steps_dev.data_ptr(), n_steps)
        lib = _lib.load()
        _lib.check(lib.tpcb_train_epoch(
            self.dm.handle, self.P.data_ptr(), self.PT.data_ptr(), self.m.data_ptr(),
            self.v.data_ptr(), C.byref(self.src.struct),
            C.byref(self.tgt.struct) if self.tgt is not None else None, C.byref(plan),
            C.byref(self.loss), C.byref(self.opt), self.hyper_dev.data_ptr(),
            self.t0_dev.data_ptr(), C.byref(self.ws.struct), self.step_loss.data_ptr(),
            self.step_cmd.data_ptr(), self.status.ptr, self.graph,
            None if profile is None else profile.ctypes.data_as(C.c_void_p),
            self.comm.handle if self.comm is not None else None,
            self.grad.data_ptr() if self.grad is not None else None,
            engine.stream_ptr()), "train_epoch")
        self.t += n_steps
        return n_steps

    def evaluate_async(self) -> None:
        """Fused forward + decode on the validation set, metrics on device."""
        with torch.cuda.stream(self.stream):
            self._evaluate_async()

    def _evaluate_async(self) -> None:
        lat = engine.run_forward(self.dm, self.P, self.valid_pk, self.valid_devfeat,
                                 self.status, self.normalizer, latents=False)[4]
        _lib.check(_lib.load().tpcb_metrics(lat.data_ptr(), self.valid_y.data_ptr(),
                                            self.valid.n_ast, self.metrics_dev.data_ptr(),
                                            engine.stream_ptr()), "metrics")

    def collect(self, n_steps: int, epoch: int):
        """One sync: per-step losses, CMD values, metrics, status."""
        with torch.cuda.stream(self.stream):
            return self._collect(n_steps, epoch)

    def _collect(self, n_steps: int, epoch: int):
        code = int(self.status.t.item())
        losses = self.step_loss[:n_steps].cpu().numpy()
        cmds = self.step_cmd[:n_steps].cpu().numpy() if self.use_cmd else np.zeros(n_steps)
        met = self.metrics_dev.cpu().numpy()
        if code not in (0, 8):  # 8 = DomainError in the validation decode
            self.status.t.zero_()
            _lib.check(code, "train", epoch)
        domain = code == 8
        if domain:
            self.status.t.zero_()
        if not np.all(np.isfinite(losses)):
            raise NonFiniteLoss(epoch)
        if domain:
            met = np.array([math.inf, math.inf, math.inf])
        return losses, cmds, met

    def tensors(self, flat: torch.Tensor | None = None) -> dict:
        self.stream.synchronize()
        return self.dm.unflatten((self.P if flat is None else flat).double().cpu().numpy())


def _rag_from_samples(samples, devices, n_leaf_max):
    from .features import CompactBatch, check_leaf_counts
    names = list(devices)
    for s in samples:
        if s.device_id not in devices:
            raise ValidationError(f"unknown device '{s.device_id}'")
    batch = CompactBatch.from_compacts([s.compact for s in samples],
                                       [devices[n] for n in names],
                                       [names.index(s.device_id) for s in samples],
                                       dtype=np.float64)
    check_leaf_counts(batch.n_leaf, n_leaf_max)
    return batch.ragged()


def _loss_from_config(config, normalizer, alpha=0.0):
    return engine.loss_struct(config.loss_mode, config.lambda_hybrid, normalizer.loss_offset,
                              alpha, config.cmd_order, config.mape_space, normalizer)


def train(config, ds, devices: dict, normalizer=None) -> TrainResult:
    """Seeded minibatch training with best-by-validation selection
    (costmodel.py:669-718)."""
    from .costmodel import CostModelParams, init_params
    from .dataset import fit_boxcox
    config.validate()
    train_samples = ds.subset("train")
    valid_samples = ds.subset("valid")
    if not train_samples or not valid_samples:
        raise EmptyDataset("train() needs non-empty train and valid splits")
    if normalizer is None:
        normalizer = fit_boxcox([s.latency_s for s in train_samples])
    train_rag = _rag_from_samples(train_samples, devices, config.n_leaf_max)
    valid_rag = _rag_from_samples(valid_samples, devices, config.n_leaf_max)
    targets = normalizer.encode(np.array([s.latency_s for s in train_samples]))
    valid_lat = np.array([s.latency_s for s in valid_samples])
    params = init_params(config)
    if config.epochs == 0:
        return TrainResult(params=params, normalizer=normalizer, log=[], best_epoch=-1,
                           best_val_mape=math.inf)
    _check_targets(config, normalizer, targets)
    loss = _loss_from_config(config, normalizer)
    if needs_large_path(config):
        from .large_training import LargeTrainer
        tr = LargeTrainer(config, params.tensors, train_rag, targets, loss, valid_rag, valid_lat,
                          normalizer)
    else:
        tr = Trainer(config, params.tensors, train_rag, targets, loss, valid_rag, valid_lat,
                     normalizer)
    return run_loop(tr, config, params, normalizer, select_best=True)


def _check_targets(config, normalizer, targets) -> None:
    """The reference's relative term rejects non-positive shifted labels
    (costmodel.py:394-396) when a batch holding one is processed; every
    training sample is visited in the first epoch, so the check runs once
    up front (the device kernels would otherwise divide by them)."""
    if config.epochs > 0 and config.loss_mode != "mse" and config.mape_space == "transformed" \
            and np.any(targets + normalizer.loss_offset <= 0):
        raise ValidationError("shifted labels must be positive")


def needs_large_path(config) -> bool:
    """True when the fused kernels cannot hold the model (e.g.
    full_reference_config): training and inference then run layer by layer
    on the tensor cores (csrc/large.cu)."""
    from .costmodel import device_model
    return not _lib.load().tpcb_forward_fits(device_model(config).handle, 64)


def run_loop(tr: Trainer, config, params, normalizer, select_best: bool) -> TrainResult:
    from .costmodel import CostModelParams
    rng = np.random.default_rng(config.seed)
    log = []
    best = None
    best_mape = math.inf
    best_epoch = -1
    for epoch in range(config.epochs):
        lr = lr_at(config, epoch)
        flat, steps = tr.plan(rng)
        n = tr.run_epoch(lr, flat, steps)
        tr.evaluate_async()
        losses, cmds, met = tr.collect(n, epoch)
        entry = EpochLog(epoch=epoch, train_loss=float(np.mean(losses)), val_mape=float(met[0]),
                         val_rmse=float(met[1]), lr=lr)
        if tr.use_cmd:
            entry.cmd = float(np.mean(cmds))
        log.append(entry)
        if select_best and met[0] < best_mape:
            best_mape, best_epoch = float(met[0]), epoch
            with torch.cuda.stream(tr.stream):
                best = tr.P.clone()
    if not select_best:
        return TrainResult(params=CostModelParams(config, tr.tensors()), normalizer=normalizer,
                           log=log, best_epoch=config.epochs - 1,
                           best_val_mape=log[-1].val_mape if log else math.inf)
    if best_epoch < 0:
        return TrainResult(params=CostModelParams(config, tr.tensors()), normalizer=normalizer,
                           log=log, best_epoch=-1, best_val_mape=math.inf)
    return TrainResult(params=CostModelParams(config, tr.tensors(best)), normalizer=normalizer,
                       log=log, best_epoch=best_epoch, best_val_mape=best_mape)


def finetune(params, source, target_inputs: list, config, devices: dict,
             normalizer) -> TrainResult:
    """Source training + CMD alignment to unlabeled target inputs
    (costmodel.py:721-780)."""
    from .features import ragged_from_encoded
    config.validate()
    train_samples = source.subset("train")
    valid_samples = source.subset("valid")
    if not train_samples or not valid_samples:
        raise EmptyDataset("finetune() needs non-empty train and valid splits")
    if config.alpha_cmd > 0 and not target_inputs:
        raise EmptyDataset("finetune() with alpha_cmd > 0 needs target inputs")
    train_rag = _rag_from_samples(train_samples, devices, config.n_leaf_max)
    valid_rag = _rag_from_samples(valid_samples, devices, config.n_leaf_max)
    targets = normalizer.encode(np.array([s.latency_s for s in train_samples]))
    valid_lat = np.array([s.latency_s for s in valid_samples])
    tgt_rag = ragged_from_encoded(target_inputs, config.n_leaf_max) if (
        config.alpha_cmd > 0 and target_inputs) else None
    alpha = config.alpha_cmd if tgt_rag is not None else 0.0
    _check_targets(config, normalizer, targets)
    loss = _loss_from_config(config, normalizer, alpha)
    if needs_large_path(config):  # e.g. full_reference_config (alpha_cmd = 1 by default)
        from .large_training import LargeTrainer
        tr = LargeTrainer(config, params.tensors, train_rag, targets, loss, valid_rag, valid_lat,
                          normalizer, target_rag=tgt_rag)
    else:
        tr = Trainer(config, params.tensors, train_rag, targets, loss, valid_rag, valid_lat,
                     normalizer, target_rag=tgt_rag)
    return run_loop(tr, config, params, normalizer, select_best=False)
