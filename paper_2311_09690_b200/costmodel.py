"""Transformer latency predictor — the reference `tpcost.costmodel` API on B200.

Same call signatures as costmodel.py (config / params / forward / backward /
losses / train / finetune / predict / checkpoints); every numeric step of the
hot path runs in libtpcb200.so:

  forward, predict, predict_batch     K1 featurize_pack → K2+K3 fused forward
  backward (+ CMD)                    K1 → train-step kernels (train.cu)
  train / finetune epochs             one native call per epoch (train.cu),
                                      optimizer in optim.cu
Host code here only validates inputs (raising the reference's exceptions
before any compute, as costmodel.py does), moves numpy arrays to and from the
device and runs the seeded host-side batch planning of costmodel.py:632-645.
"""

from __future__ import annotations

import hashlib
import io
import json
import math
import threading
import zipfile
from dataclasses import asdict, dataclass, replace

import numpy as np
import torch

from . import _lib, engine
from .dataset import BoxCoxNormalizer, fit_boxcox
from .errors import (CheckpointError, DimensionMismatch, DomainError, EmptyBatch,
                     EmptyDataset, EmptySet, NonFiniteLoss, UnsupportedConfig, ValidationError)
from .features import (N_ENTRY, CompactAst, CompactBatch, DeviceSpec, EncodedInput,
                       check_leaf_counts, device_vector, encode_input, ragged_from_encoded)

DEVICE_FEATURES = 6


# ---------------------------------------------------------------------------
# configuration / parameters (costmodel.py:36-150)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class CostModelConfig:
    d_model: int = 64
    n_layers: int = 2
    n_heads: int = 2
    d_ff: int = 128
    d_embed: int = 32
    d_device: int = 16
    decoder_dims: tuple = (64, 64)
    n_leaf_max: int = 16
    lambda_hybrid: float = 1e-3
    alpha_cmd: float = 0.0
    cmd_order: int = 5
    lr: float = 1e-3
    weight_decay: float = 0.0
    optimizer: str = "adam"
    lr_schedule: str = "constant"
    batch_size: int = 64
    epochs: int = 300
    seed: int = 0
    loss_mode: str = "hybrid"
    mape_space: str = "transformed"

    def validate(self) -> None:
        if self.d_model % self.n_heads != 0:
            raise ValidationError("d_model must be divisible by n_heads")
        for a in ("d_model", "n_layers", "n_heads", "d_ff", "d_embed", "d_device",
                  "n_leaf_max", "batch_size"):
            if getattr(self, a) < 1:
                raise ValidationError(f"{a} must be >= 1")
        if self.epochs < 0:
            raise ValidationError("epochs must be >= 0")
        if any(w < 1 for w in self.decoder_dims):
            raise ValidationError("decoder widths must be >= 1")
        if self.lr <= 0 or self.lambda_hybrid < 0 or self.alpha_cmd < 0:
            raise ValidationError("lr must be > 0; loss coefficients >= 0")
        if self.cmd_order < 1:
            raise ValidationError("cmd_order must be >= 1")
        if self.optimizer not in ("adam", "sgd"):
            raise ValidationError(f"unknown optimizer '{self.optimizer}'")
        if self.lr_schedule not in ("constant", "cyclic"):
            raise ValidationError(f"unknown lr_schedule '{self.lr_schedule}'")
        if self.loss_mode not in ("hybrid", "mse", "mape"):
            raise ValidationError(f"unknown loss_mode '{self.loss_mode}'")
        if self.mape_space not in ("original", "transformed"):
            raise ValidationError(f"unknown mape_space '{self.mape_space}'")


def desk_config(**overrides) -> CostModelConfig:
    return replace(CostModelConfig(), **overrides)


def full_reference_config() -> CostModelConfig:
    return CostModelConfig(d_model=716, n_layers=11, n_heads=4, d_ff=985, d_embed=69,
                           d_device=64, decoder_dims=(930, 930, 930), n_leaf_max=16,
                           lambda_hybrid=1e-3, alpha_cmd=1.0, lr=1.68e-5, weight_decay=0.0013,
                           optimizer="adam", lr_schedule="cyclic", batch_size=600)


@dataclass
class CostModelParams:
    config: CostModelConfig
    tensors: dict

    def n_params(self) -> int:
        return sum(t.size for t in self.tensors.values())

    def copy(self) -> "CostModelParams":
        return CostModelParams(self.config, {k: v.copy() for k, v in self.tensors.items()})


def _xavier(rng, fan_in, fan_out):
    bound = math.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-bound, bound, size=(fan_in, fan_out))


def init_params(config: CostModelConfig) -> CostModelParams:
    """Seeded Xavier-uniform init; LN gains 1, biases 0; same tensor creation
    order — hence bit-identical tensors — as costmodel.py:116-150."""
    config.validate()
    rng = np.random.default_rng(config.seed)
    t: dict = {}
    d = config.d_model

    def lin(name, fi, fo):
        t[f"{name}.W"] = _xavier(rng, fi, fo)
        t[f"{name}.b"] = np.zeros(fo)

    lin("input", N_ENTRY, d)
    for i in range(config.n_layers):
        p = f"enc{i}"
        for w in ("Wq", "Wk", "Wv", "Wo"):
            t[f"{p}.attn.{w}"] = _xavier(rng, d, d)
        for b in ("bq", "bk", "bv", "bo"):
            t[f"{p}.attn.{b}"] = np.zeros(d)
        t[f"{p}.ln1.g"] = np.ones(d)
        t[f"{p}.ln1.b"] = np.zeros(d)
        lin(f"{p}.ffn.h", d, config.d_ff)
        lin(f"{p}.ffn.o", config.d_ff, d)
        t[f"{p}.ln2.g"] = np.ones(d)
        t[f"{p}.ln2.b"] = np.zeros(d)
    for L in range(1, config.n_leaf_max + 1):
        lin(f"leaf_embed.{L}", L * d, config.d_embed)
    lin("dev.hidden", DEVICE_FEATURES, config.d_device)
    lin("dev.proj", config.d_device, config.d_embed)
    w = config.d_embed
    for i, h in enumerate(config.decoder_dims):
        lin(f"dec.{i}", w, h)
        w = h
    lin("dec.out", w, 1)
    return CostModelParams(config=config, tensors=t)


@dataclass
class LatentBatch:
    z_x: np.ndarray
    z_v: np.ndarray
    z: np.ndarray


# ---------------------------------------------------------------------------
# device model cache
# ---------------------------------------------------------------------------

_MODELS: dict = {}


def device_model(config: CostModelConfig) -> engine.DeviceModel:
    key = (config.d_model, config.n_layers, config.n_heads, config.d_ff, config.d_embed,
           config.d_device, tuple(config.decoder_dims), config.n_leaf_max)
    dm = _MODELS.get(key)
    if dm is None:
        dm = _MODELS[key] = engine.DeviceModel(config)
    return dm


class Predictor:
    """Device-resident model: flat fp32 parameters + the model handle.
    The bulk inference entry point (`forward_batch`) of the GPU path."""

    def __init__(self, params: CostModelParams, rows_per_tile: int | None = None,
                 precision: str = "fp32",
                 path: str = "auto"):
        """precision "fp32": the parity mode (FP32 FFMA, decoded latency within
        1e-3 of the float64 reference); "bf16": encoder GEMMs on the tcgen05
        tensor cores with bf16 operands and fp32 accumulation (desk-shaped
        models; packs 128-row tiles), accuracy stated in DESIGN.md.
        path "auto" | "fused" | "large": the layer-by-layer tensor-core path
        (csrc/large.cu) is taken automatically when the fused kernels cannot
        hold the model; "large" forces it (tests)."""
        if path not in ("auto", "fused", "large"):
            raise ValidationError(f"unknown path {path!r}")
        if precision not in ("fp32", "bf16"):
            raise ValidationError(f"unknown precision {precision!r}")
        self.config = params.config
        self.dm = device_model(params.config)
        self.params = self.dm.upload(params.tensors)
        self.precision = precision
        if precision == "bf16":
            self.R = 128
        elif rows_per_tile is None:  # 128 for desk shapes (forward_f32.cu), else 64
            self.R = int(_lib.load().tpcb_forward_rows(self.dm.handle))
        else:
            self.R = rows_per_tile
        self.status = engine.Status(self.params.device)
        # configs the fused one-CTA-per-tile kernels cannot hold (e.g.
        # full_reference_config) run layer by layer on the tensor cores
        # (3xTF32 GEMMs, fp32-accumulate parity accuracy) in either precision
        self.large = None
        fits = bool(_lib.load().tpcb_forward_fits(self.dm.handle, self.R))
        if path == "fused" and not fits:
            raise UnsupportedConfig("the fused forward cannot hold this model")
        if path == "large" or not fits:
            self.large = engine.LargePath(self.dm, self.params)

    def tensors(self) -> dict:
        return self.dm.unflatten(self.params.double().cpu().numpy())

    def forward_device(self, rows, ordering, leaf_off, devfeat, n_ast, encoded, norm=None,
                       latents=True, theta=engine.THETA_DEFAULT, n_leaf=None):
        """n_leaf: host leaf counts (the large path plans its buckets on the
        host; read back from leaf_off when not given)."""
        pk = engine.pack(rows, ordering, leaf_off, n_ast, self.config.n_leaf_max, encoded,
                         self.status, self.R, theta)
        if self.large is not None:
            if n_leaf is None:
                n_leaf = np.diff(leaf_off.cpu().numpy())
            return self.large.forward(pk, n_leaf, devfeat, self.status, norm, latents)
        return engine.run_forward(self.dm, self.params, pk, devfeat, self.status, norm, latents,
                                  self.precision)

    def forward_ragged(self, rag: engine.RaggedHost, norm=None, latents=True):
        if rag.n_ast == 0:
            raise EmptyBatch("forward needs at least one input")
        check_leaf_counts(rag.n_leaf, self.config.n_leaf_max)
        rows, ordering, leaf_off, devfeat = engine.upload_ragged(rag)
        out = self.forward_device(rows, ordering, leaf_off, devfeat, rag.n_ast, rag.encoded,
                                  norm, latents, n_leaf=rag.n_leaf)
        self.status.check("forward")
        return out

    # ASTs per pipelined chunk of forward_batch (host↔device copies of chunk
    # i+1 overlap the featurize + forward of chunk i)
    CHUNK = 1 << 18

    def forward_batch(self, batch: CompactBatch, normalizer=None, latents=False):
        """Bulk path: raw compact ASTs in, (pred, z_x, z_v, z, latency) out.

        Large batches run as a pipeline of CHUNK-AST pieces on two streams:
        the H2D copy of a piece's rows / orderings / leaf counts / device
        indices overlaps the previous piece's K1 + forward, leaf offsets and
        device features are formed on the device, results come back with
        async D2H copies into pinned buffers.  Per-AST results do not depend
        on the batching (every kernel is per AST / per token row), so the
        output equals the one-shot path bit for bit.  Host arrays in pinned
        memory (e.g. views of `torch.Tensor.pin_memory()`) get the overlap;
        pageable arrays still work, with the copies serialised."""
        n = batch.n_ast
        if n == 0:
            raise EmptyBatch("forward needs at least one input")
        if self.large is not None or n <= self.CHUNK:
            pred, zx, zv, z, lat = self.forward_ragged(batch.ragged(), normalizer, latents)
            cpu = lambda t: None if t is None else t.cpu().numpy()  # noqa: E731
            return cpu(pred), cpu(zx), cpu(zv), cpu(z), cpu(lat)
        return self._forward_pipelined(batch, normalizer, latents)

    def _pipe_state(self):
        """Per-thread pipeline state (buffers + copy stream): concurrent
        forward_batch calls on one Predictor from different threads never
        share a staging buffer."""
        tls = self.__dict__.get("_tls")
        if tls is None:
            tls = self.__dict__.setdefault("_tls", threading.local())
        if not hasattr(tls, "bufs"):
            tls.bufs = {}
            tls.copy = None
        return tls

    def _buf(self, name, numel, dtype, device=None):
        """Cached pipeline buffer (device, or pinned host when device is None),
        grown on demand; every call synchronises before returning, so a buffer
        is never resized under in-flight work."""
        cache = self._pipe_state().bufs
        buf = cache.get(name)
        if buf is None or buf.numel() < numel or buf.dtype != dtype:
            buf = (torch.empty(max(numel, 1), dtype=dtype, device=device) if device is not None
                   else torch.empty(max(numel, 1), dtype=dtype, pin_memory=True))
            cache[name] = buf
        return buf[:numel]

    def _forward_pipelined(self, batch: CompactBatch, normalizer, latents):
        n = batch.n_ast
        n_leaf = np.ascontiguousarray(batch.n_leaf, dtype=np.int64)
        dev = self.params.device
        table = torch.from_numpy(np.stack([device_vector(d) for d in batch.devices])
                                 .astype(np.float32)).to(dev)

        def t(a, small=False):
            # a copy from pageable memory blocks the host until the copy stream
            # drains, which serialises the pipeline: small arrays (counts,
            # orderings, device indices) are staged into pinned memory once;
            # the rows are used as given (pin them to get the overlap)
            x = torch.from_numpy(np.ascontiguousarray(a))
            return x.pin_memory() if small and not x.is_pinned() else x
        rows_h = t(batch.vectors)
        ord_h = t(np.asarray(batch.ordering, dtype=np.int32), small=True)
        nl_h = t(n_leaf, small=True)
        one_dev = len(batch.devices) == 1  # every AST on device 0: no index upload
        di_h = None if one_dev else t(np.asarray(batch.device_index, dtype=np.int32), small=True)
        # a short first piece fills the pipeline sooner
        bounds = [0] + list(range(min(n, self.CHUNK // 4), n, self.CHUNK)) + [n]
        tok = np.add.reduceat(n_leaf, bounds[:-1])  # tokens per piece
        cap_tok, cap_ast = int(tok.max()), int(np.diff(bounds).max())
        F = rows_h.shape[1]
        # two sets of device input buffers reused across pieces and calls (fresh
        # allocations per piece, held by the side stream, made the caching
        # allocator fall back to cudaMalloc / cudaFree — device-wide syncs)
        ins = [(self._buf(f"rows{k}", cap_tok * F, rows_h.dtype, dev),
                self._buf(f"ord{k}", cap_tok, torch.int32, dev),
                self._buf(f"nl{k}", cap_ast, torch.int64, dev),
                None if one_dev else self._buf(f"di{k}", cap_ast, torch.int32, dev))
               for k in range(2)]
        de, ddev = self.config.d_embed, self.config.d_device
        # outputs: fresh pinned arrays handed to the caller (no host copy; the
        # caching host allocator recycles them once the caller drops them)
        pinned = lambda *shape, dt=torch.float32: torch.empty(  # noqa: E731
            shape, dtype=dt, pin_memory=True)
        out_pred = pinned(n)
        out_lat = pinned(n, dt=torch.float64) if normalizer is not None else None
        outs_lat = [pinned(n, w) for w in (de, ddev, de)] if latents else None
        compute = torch.cuda.current_stream(dev)
        st = self._pipe_state()
        if st.copy is None:
            st.copy = torch.cuda.Stream(device=dev)
        copy = st.copy
        free = [None, None]  # compute finished with input buffer set k
        keep = []
        tb = 0
        for i, (a, b) in enumerate(zip(bounds[:-1], bounds[1:])):
            nl_c = n_leaf[a:b]
            if nl_c.min() < 1 or nl_c.max() > self.config.n_leaf_max:
                compute.synchronize()  # pieces already queued finish; nothing is returned
                check_leaf_counts(n_leaf, self.config.n_leaf_max)  # raises, global index
            if one_dev and np.any(batch.device_index[a:b]):  # as table[device_index] would
                compute.synchronize()
                raise IndexError("device index out of range for a batch with one device")
            ta, tb = tb, tb + int(tok[i])
            k = i & 1
            rows_d, ord_d, nl_d, di_d = ins[k]
            rows = rows_d[:(tb - ta) * F].view(tb - ta, F)
            ordering, nl = ord_d[:tb - ta], nl_d[:b - a]
            di = None if one_dev else di_d[:b - a]
            with torch.cuda.stream(copy):  # H2D of this piece (async from pinned memory)
                if free[k] is not None:
                    copy.wait_event(free[k])
                rows.copy_(rows_h[ta:tb], non_blocking=True)
                ordering.copy_(ord_h[ta:tb], non_blocking=True)
                nl.copy_(nl_h[a:b], non_blocking=True)
                if di is not None:
                    di.copy_(di_h[a:b], non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(copy)
            compute.wait_event(ready)
            leaf_off = torch.zeros(b - a + 1, dtype=torch.int64, device=dev)
            torch.cumsum(nl, 0, out=leaf_off[1:])
            devfeat = table[:1].expand(b - a, -1).contiguous() if one_dev else \
                table.index_select(0, di.long())
            pred, zx, zv, z, lat = self.forward_device(rows, ordering, leaf_off, devfeat, b - a,
                                                       False, normalizer, latents)
            free[k] = torch.cuda.Event()
            free[k].record(compute)
            out_pred[a:b].copy_(pred, non_blocking=True)
            if out_lat is not None:
                out_lat[a:b].copy_(lat, non_blocking=True)
            if latents:
                for o, v in zip(outs_lat, (zx, zv, z)):
                    o[a:b].copy_(v, non_blocking=True)
            keep.append((pred, zx, zv, z, lat))  # alive until the D2H copies ran
        compute.synchronize()
        self.status.check("forward")
        res = (out_pred.numpy(),) + (tuple(o.numpy() for o in outs_lat) if latents
                                     else (None, None, None))
        return res + (out_lat.numpy() if out_lat is not None else None,)


def forward(params: CostModelParams, inputs: list) -> tuple:
    """Predictions (model space) and latents (costmodel.py:265-269)."""
    if not inputs:
        raise EmptyBatch("forward needs at least one input")
    rag = ragged_from_encoded(inputs, params.config.n_leaf_max)
    p = Predictor(params)
    pred, zx, zv, z, _ = p.forward_ragged(rag)
    f64 = lambda t: t.double().cpu().numpy()  # noqa: E731
    return f64(pred), LatentBatch(z_x=f64(zx), z_v=f64(zv), z=f64(z))


def predict(params: CostModelParams, compact: CompactAst, device: DeviceSpec,
            normalizer: BoxCoxNormalizer) -> float:
    """Latency in seconds for one program (costmodel.py:795-800)."""
    normalizer._check()
    batch = CompactBatch.from_compacts([compact], device, dtype=np.float64)
    _, _, _, _, lat = Predictor(params).forward_batch(batch, normalizer)
    return float(lat[0])


def predict_batch(params: CostModelParams, inputs: list,
                  normalizer: BoxCoxNormalizer) -> np.ndarray:
    """Decoded latencies for encoded inputs (costmodel.py:803-806)."""
    normalizer._check()
    if not inputs:
        raise EmptyBatch("forward needs at least one input")
    rag = ragged_from_encoded(inputs, params.config.n_leaf_max)
    _, _, _, _, lat = Predictor(params).forward_ragged(rag, normalizer, latents=False)
    return lat.cpu().numpy()


# ---------------------------------------------------------------------------
# losses / metrics (costmodel.py:343-355, 489-508, 577-591)
# ---------------------------------------------------------------------------

def loss_pretrain(pred, y, lambda_hybrid: float = 1e-3) -> float:
    pred = np.asarray(pred, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if pred.size == 0:
        raise EmptyBatch("loss needs at least one sample")
    if pred.shape != y.shape:
        raise ValidationError("pred and y must have equal length")
    if np.any(y <= 0):
        raise ValidationError("labels must be positive for the relative term")
    diff = pred - y
    return float(np.mean(diff ** 2) + lambda_hybrid * np.mean(np.abs(diff) / y))


def metrics(pred, y) -> dict:
    pred = np.asarray(pred, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if pred.size == 0:
        raise EmptyBatch("metrics need at least one sample")
    if pred.shape != y.shape:
        raise ValidationError("pred and y must have equal length")
    if np.any(y <= 0):
        raise ValidationError("labels must be positive")
    diff = pred - y
    rel = diff / y
    return {"mape": float(np.mean(np.abs(rel))), "rmse": float(math.sqrt(np.mean(diff ** 2))),
            "mspe": float(np.mean(rel ** 2))}


def encode_dataset(samples, devices: dict) -> list:
    out = []
    for s in samples:
        if s.device_id not in devices:
            raise ValidationError(f"unknown device '{s.device_id}'")
        out.append(encode_input(s.compact, devices[s.device_id]))
    return out


# ---------------------------------------------------------------------------
# CMD (costmodel.py:489-508, 783-788)
# ---------------------------------------------------------------------------

def _cmd_device(zs, zt, k: int, want_grad: bool):
    zs = np.atleast_2d(np.asarray(zs, dtype=np.float64))
    zt = np.atleast_2d(np.asarray(zt, dtype=np.float64))
    if zs.shape[0] == 0 or zt.shape[0] == 0:
        raise EmptySet("cmd needs non-empty sets")
    if zs.shape[1] != zt.shape[1]:
        raise DimensionMismatch(f"column mismatch: {zs.shape[1]} vs {zt.shape[1]}")
    engine._need_cuda()
    z = torch.from_numpy(np.ascontiguousarray(np.vstack([zs, zt]))).cuda()
    val = torch.zeros(1, dtype=torch.float64, device=z.device)
    grad = torch.empty_like(z) if want_grad else None
    cmd_device_z(z, zs.shape[0], zt.shape[0], int(k), val, grad)
    value = float(val.item())
    if not want_grad:
        return value
    g = grad.cpu().numpy()
    return value, g[:zs.shape[0]], g[zs.shape[0]:]


CMD_GRID_ROWS = 16384  # at or above: the multi-block HBM-streaming kernels


def cmd_device_z(z: torch.Tensor, ns: int, nt: int, k: int, val: torch.Tensor,
                 grad: torch.Tensor | None = None) -> None:
    """CMD of device rows z = [zs; zt] (f32/f64) into val[0] (+ grad):
    one CTA for small sets (the in-step size), the grid kernels for large
    ones (cmd_between over whole datasets)."""
    lib = engine._lib.load()
    is64 = 1 if z.dtype == torch.float64 else 0
    de = int(z.shape[1])
    if ns + nt >= CMD_GRID_ROWS and de <= 128:
        ws = torch.empty(int(lib.tpcb_cmd_grid_ws(ns, nt, de, k)), dtype=torch.uint8,
                         device=z.device)
        engine._lib.check(lib.tpcb_cmd_grid(z.data_ptr(), is64, ns, nt, de, k, val.data_ptr(),
                                            engine.dptr(grad), ws.data_ptr(), ws.numel(),
                                            engine.stream_ptr()), "cmd")
    else:
        engine._lib.check(lib.tpcb_cmd(z.data_ptr(), is64, ns, nt, de, k, val.data_ptr(),
                                       engine.dptr(grad), engine.stream_ptr()), "cmd")


def cmd(zs, zt, k: int = 5) -> float:
    """Central moment discrepancy between two sample sets, fp64 on the GPU."""
    return _cmd_device(zs, zt, k, False)


def cmd_grad(zs, zt, k: int = 5):
    """(value, dCMD/dzs, dCMD/dzt) — `_cmd_forward_backward` (costmodel.py:426-486)."""
    return _cmd_device(zs, zt, k, True)


def loss_finetune(pred, y, zs, zt, lambda_hybrid: float = 1e-3, alpha_cmd: float = 1.0,
                  k: int = 5) -> float:
    return loss_pretrain(pred, y, lambda_hybrid) + alpha_cmd * cmd(zs, zt, k)


def cmd_between(params: CostModelParams, source_inputs: list, target_inputs: list,
                k: int = 5) -> float:
    """CMD between the aggregated latents of two full input sets."""
    _, ls = forward(params, source_inputs)
    _, lt = forward(params, target_inputs)
    return cmd(ls.z, lt.z, k)


# ---------------------------------------------------------------------------
# backward (costmodel.py:511-570)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class LossSpec:
    mode: str = "hybrid"
    lambda_hybrid: float = 1e-3
    alpha_cmd: float = 0.0
    cmd_order: int = 5
    offset: float = 0.0
    mape_space: str = "transformed"
    normalizer: BoxCoxNormalizer | None = None


def _check_loss(loss: LossSpec, targets: np.ndarray) -> None:
    if loss.mode not in ("hybrid", "mse", "mape"):
        raise ValidationError(f"unknown loss mode '{loss.mode}'")
    if loss.mode == "mse":
        return
    if loss.mape_space == "original":
        if loss.normalizer is None:
            raise ValidationError("original-space relative loss needs a fitted normalizer")
        loss.normalizer._check()
        t = np.asarray(targets) * loss.normalizer.t_std + loss.normalizer.t_mean
        if abs(loss.normalizer.lambda_bc) >= 1e-9 and np.any(loss.normalizer.lambda_bc * t + 1.0 <= 0):
            raise DomainError("no positive preimage: lambda*t + 1 <= 0")
    elif np.any(np.asarray(targets) + loss.offset <= 0):
        raise ValidationError("shifted labels must be positive")


def _loss_struct(loss: LossSpec):
    return engine.loss_struct(loss.mode, loss.lambda_hybrid, loss.offset, loss.alpha_cmd,
                              loss.cmd_order, loss.mape_space, loss.normalizer)


def backward(params: CostModelParams, batch: list, targets, loss: LossSpec,
             target_batch: list | None = None, *, wgrad_tc: bool = False):
    """Loss value and d(objective)/d(every parameter) (costmodel.py:529-570),
    computed by the fused train-step kernels; with alpha_cmd > 0 and a target
    batch the CMD term couples both forward passes.  wgrad_tc=True
    (desk shapes, no CMD): the encoder weight gradients as tcgen05 3xTF32
    GEMMs over the batch's token rows (csrc/wgrad.cu) instead of the
    per-sample slots"""
    targets = np.asarray(targets, dtype=np.float64)
    if not batch:
        raise EmptyBatch("forward needs at least one input")
    cfg = params.config
    rag = ragged_from_encoded(batch, cfg.n_leaf_max)
    if targets.shape != (len(batch),):
        raise ValidationError("batch and targets must have equal length")
    _check_loss(loss, targets)
    use_cmd = loss.alpha_cmd > 0.0 and target_batch is not None
    trag = None
    if use_cmd:
        if not target_batch:
            raise EmptyBatch("forward needs at least one input")
        trag = ragged_from_encoded(target_batch, cfg.n_leaf_max)
    dm = device_model(cfg)
    P = dm.upload(params.tensors)
    PT = torch.empty_like(P)
    engine.transpose_params(dm, P, PT)
    st = engine.Status(P.device)
    src = engine.DeviceSamples(rag, cfg.n_leaf_max, st, y=targets)
    tgt = engine.DeviceSamples(trag, cfg.n_leaf_max, st) if use_cmd else None
    l_cap = max(int(rag.n_leaf.max()), int(trag.n_leaf.max()) if trag is not None else 1)
    ws = engine.TrainWorkspace(dm, src.n + (tgt.n if tgt else 0), l_cap=l_cap, overlap=False,
                               wgrad_tc=wgrad_tc)
    grad, pred = engine.run_backward(dm, P, PT, src, tgt, _loss_struct(loss), ws, st)
    st.check("backward")
    sc = ws.scalars.cpu().numpy()
    value = float(sc[1])
    cmd_value = float(sc[0]) if use_cmd else 0.0
    grads = dm.unflatten(grad.double().cpu().numpy())
    if not math.isfinite(value):
        raise NonFiniteLoss(-1)
    return value, grads, {"pred": pred.double().cpu().numpy(), "cmd": cmd_value}


# ---------------------------------------------------------------------------
# training loops (costmodel.py:598-780) — device resident, see training.py
# ---------------------------------------------------------------------------

from .training import EpochLog, TrainResult, Trainer, epoch_batches, finetune, lr_at, train  # noqa: E402,F401


# ---------------------------------------------------------------------------
# checkpoints (costmodel.py:902-956) — same file format
# ---------------------------------------------------------------------------

_CHECKPOINT_VERSION = 1


def _tensor_checksum(tensors: dict) -> str:
    h = hashlib.sha256()
    for name in sorted(tensors):
        arr = np.ascontiguousarray(tensors[name], dtype=np.float64)
        h.update(name.encode())
        h.update(str(arr.shape).encode())
        h.update(arr.tobytes())
    return h.hexdigest()


def save_checkpoint(path, params: CostModelParams, normalizer=None) -> None:
    cfg = asdict(params.config)
    cfg["decoder_dims"] = list(cfg["decoder_dims"])
    meta = {"version": _CHECKPOINT_VERSION, "config": cfg,
            "normalizer": asdict(normalizer) if normalizer is not None else None,
            "checksum": _tensor_checksum(params.tensors)}
    meta_bytes = np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8)
    buf = io.BytesIO()
    np.savez(buf, __meta__=meta_bytes, **params.tensors)
    with open(path, "wb") as f:
        f.write(buf.getvalue())


def load_checkpoint(path):
    try:
        with np.load(path) as data:
            if "__meta__" not in data:
                raise CheckpointError("missing metadata block")
            meta = json.loads(bytes(data["__meta__"]).decode())
            if meta.get("version") != _CHECKPOINT_VERSION:
                raise CheckpointError(f"unsupported version {meta.get('version')}")
            tensors = {n: np.asarray(data[n], dtype=np.float64)
                       for n in data.files if n != "__meta__"}
    except (ValueError, KeyError, OSError, json.JSONDecodeError, zipfile.BadZipFile) as e:
        raise CheckpointError(f"cannot read checkpoint: {e}") from e
    if _tensor_checksum(tensors) != meta["checksum"]:
        raise CheckpointError("checksum mismatch: corrupt checkpoint")
    cfg = dict(meta["config"])
    cfg["decoder_dims"] = tuple(cfg["decoder_dims"])
    params = CostModelParams(config=CostModelConfig(**cfg), tensors=tensors)
    norm = BoxCoxNormalizer(**meta["normalizer"]) if meta["normalizer"] is not None else None
    return params, norm
