"""Device-side runtime: model handles, packed batches and kernel launches.

PyTorch is used only as the device allocator / stream provider; all compute
is in libtpcb200.so (see include/tpcb200.h).  Everything here is
stream-ordered on torch's current stream; `sync_status` is the only place
that synchronises, to turn the device status word into the reference's
exceptions.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import errors as E

THETA_DEFAULT = 10000.0


def _need_cuda():
    if not torch.cuda.is_available():
        raise E.CudaError("a CUDA device is required (no CPU fallback)")
    _lib.load()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def dptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def pe_denominators(theta: float = THETA_DEFAULT) -> np.ndarray:
    """θ^(2δ/24), δ=0..11 — computed with numpy exactly as features.py:257-258
    so the device divides by bit-identical denominators."""
    if theta <= 0:
        raise E.ValidationError("theta must be > 0")
    return float(theta) ** (2.0 * np.arange(12, dtype=np.float64) / 24)


class Status:
    """Device status word shared by a sequence of launches."""

    def __init__(self, device):
        self.t = torch.zeros(1, dtype=torch.int32, device=device)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def check(self, what: str, epoch: int = -1) -> None:
        code = int(self.t.item())  # synchronises the stream
        if code:
            self.t.zero_()
            _lib.check(code, what, epoch)


# ---------------------------------------------------------------------------
# model handle + flat parameter vector
# ---------------------------------------------------------------------------

class DeviceModel:
    """tpcb_model handle + canonical layout of the flat fp32 parameter vector."""

    def __init__(self, cfg):
        _need_cuda()
        lib = _lib.load()
        c = _lib.Config()
        c.d_model, c.n_layers, c.n_heads = cfg.d_model, cfg.n_layers, cfg.n_heads
        c.d_ff, c.d_embed, c.d_device = cfg.d_ff, cfg.d_embed, cfg.d_device
        dec = tuple(cfg.decoder_dims)
        if len(dec) > _lib.MAX_DEC:
            raise E.UnsupportedConfig("too many decoder layers")
        c.n_dec = len(dec)
        for i, w in enumerate(dec):
            c.dec[i] = w
        c.n_leaf_max = cfg.n_leaf_max
        h = C.c_void_p()
        _lib.check(lib.tpcb_model_create(C.byref(c), C.byref(h)), "model_create")
        self.handle = h
        self.cfg = cfg
        self.n_params = int(lib.tpcb_model_param_count(h))
        self.layout: dict[str, tuple[int, tuple]] = {}
        buf = C.create_string_buffer(128)
        off, r, cc = C.c_int64(), C.c_int32(), C.c_int32()
        for i in range(lib.tpcb_model_tensor_count(h)):
            lib.tpcb_model_tensor_info(h, i, buf, 128, C.byref(off), C.byref(r), C.byref(cc))
            shape = (r.value, cc.value) if cc.value else (r.value,)
            self.layout[buf.value.decode()] = (off.value, shape)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _lib.load().tpcb_model_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def flatten(self, tensors: dict[str, np.ndarray]) -> np.ndarray:
        flat = np.zeros(self.n_params, dtype=np.float64)
        for name, (o, shape) in self.layout.items():
            t = np.asarray(tensors[name], dtype=np.float64)
            if t.shape != shape:
                raise E.ValidationError(f"tensor {name}: shape {t.shape} != {shape}")
            flat[o:o + t.size] = t.ravel()
        return flat

    def unflatten(self, flat: np.ndarray) -> dict[str, np.ndarray]:
        out = {}
        for name, (o, shape) in self.layout.items():
            n = int(np.prod(shape))
            out[name] = np.asarray(flat[o:o + n], dtype=np.float64).reshape(shape).copy()
        return out

    def upload(self, tensors: dict[str, np.ndarray], device="cuda") -> torch.Tensor:
        return torch.from_numpy(self.flatten(tensors).astype(np.float32)).to(device)

    def slice_of(self, name: str) -> slice:
        o, shape = self.layout[name]
        return slice(o, o + int(np.prod(shape)))


# ---------------------------------------------------------------------------
# ragged batch → packed tiles (K1)
# ---------------------------------------------------------------------------

@dataclass
class RaggedHost:
    """Host SoA of a batch of compact ASTs (or encoded matrices)."""
    rows: np.ndarray        # (n_tok, 24) float32/float64
    ordering: np.ndarray    # (n_tok,) int32 (unused when encoded=True)
    n_leaf: np.ndarray      # (n_ast,) int64
    devfeat: np.ndarray     # (n_ast, 6) float32
    encoded: bool           # rows already carry the PE

    @property
    def n_ast(self) -> int:
        return int(self.n_leaf.shape[0])

    @property
    def n_tok(self) -> int:
        return int(self.rows.shape[0])


class PackedBatch:
    """Device buffers of the packed fixed-stride layout (tpcb_packed)."""

    def __init__(self, n_ast: int, n_tok: int, n_leaf_max: int, R: int, device):
        lib = _lib.load()
        ntm, ws = C.c_int32(), C.c_size_t()
        _lib.check(lib.tpcb_pack_sizes(n_ast, n_tok, n_leaf_max, R, C.byref(ntm), C.byref(ws)),
                   "pack_sizes")
        self.n_ast, self.n_tok, self.R, self.n_leaf_max = n_ast, n_tok, R, n_leaf_max
        self.n_tiles_max = ntm.value
        i32 = dict(dtype=torch.int32, device=device)
        self.x = torch.empty(ntm.value * R * _lib.FEAT_PAD, dtype=torch.float32, device=device)
        self.row_ast = torch.empty(ntm.value * R, **i32)
        self.tile_L = torch.empty(ntm.value, **i32)
        self.tile_first = torch.empty(ntm.value, **i32)
        self.tile_count = torch.empty(ntm.value, **i32)
        self.perm = torch.empty(max(n_ast, 1), **i32)
        self.ast_row = torch.empty(max(n_ast, 1), **i32)
        self.bucket_off = torch.empty(n_leaf_max + 2, **i32)
        self.n_tiles = torch.zeros(1, **i32)
        self.ws = torch.empty(max(ws.value, 4), dtype=torch.uint8, device=device)
        s = _lib.Packed()
        s.rows_per_tile, s.n_tiles_max = R, ntm.value
        for f in ("x", "row_ast", "tile_L", "tile_first", "tile_count", "perm", "ast_row",
                  "bucket_off", "n_tiles"):
            setattr(s, f, getattr(self, f).data_ptr())
        self.struct = s


def upload_ragged(rag: RaggedHost, device="cuda"):
    rows = torch.from_numpy(np.ascontiguousarray(rag.rows)).to(device, non_blocking=True)
    ordering = torch.from_numpy(np.ascontiguousarray(rag.ordering, dtype=np.int32)).to(device)
    off = np.zeros(rag.n_ast + 1, dtype=np.int64)
    np.cumsum(rag.n_leaf, out=off[1:])
    leaf_off = torch.from_numpy(off).to(device)
    devfeat = torch.from_numpy(np.ascontiguousarray(rag.devfeat, dtype=np.float32)).to(device)
    return rows, ordering, leaf_off, devfeat


def pack(rows: torch.Tensor, ordering: torch.Tensor, leaf_off: torch.Tensor, n_ast: int,
         n_leaf_max: int, encoded: bool, status: Status, R: int = 64,
         theta: float = THETA_DEFAULT, out: PackedBatch | None = None) -> PackedBatch:
    """Run K1 on device-resident ragged rows (into `out` when given: same
    buffers, so captured graphs that read them stay valid)."""
    lib = _lib.load()
    n_tok = int(rows.shape[0])
    if out is not None and (out.n_ast, out.n_tok, out.n_leaf_max) == (n_ast, n_tok, n_leaf_max):
        pk, R = out, out.R
    else:
        pk = PackedBatch(n_ast, n_tok, n_leaf_max, R, rows.device)
    den = None if encoded else pe_denominators(theta)
    den_p = None if den is None else den.ctypes.data_as(C.c_void_p)
    is64 = 1 if rows.dtype == torch.float64 else 0
    if rows.dtype not in (torch.float32, torch.float64):
        raise E.ValidationError("leaf vectors must be float32 or float64")
    _lib.check(lib.tpcb_featurize_pack(rows.data_ptr(), is64, ordering.data_ptr(),
                                       leaf_off.data_ptr(), n_ast, n_tok, n_leaf_max, den_p,
                                       pk.ws.data_ptr(), pk.ws.numel(), C.byref(pk.struct),
                                       status.ptr, stream_ptr()), "featurize_pack")
    return pk


def boxcox_struct(norm) -> _lib.BoxCox:
    b = _lib.BoxCox()
    if norm is None:
        b.enabled = 0
        return b
    b.lambda_bc, b.shift = float(norm.lambda_bc), float(norm.shift)
    b.t_mean, b.t_std = float(norm.t_mean), float(norm.t_std)
    b.enabled = 1
    return b


def run_forward(dm: DeviceModel, params: torch.Tensor, pk: PackedBatch, devfeat: torch.Tensor,
                status: Status, norm=None, latents: bool = True, precision: str = "fp32"):
    """Launch the fused forward; returns device tensors (pred, z_x, z_v, z, lat).
    precision "fp32": FP32 parity mode (tpcb_forward); "bf16": encoder GEMMs on
    the tcgen05 tensor cores (tpcb_forward_bf16; desk config, 128-row tiles)."""
    lib = _lib.load()
    n = pk.n_ast
    dev = params.device
    pred = torch.empty(n, dtype=torch.float32, device=dev)
    zx = torch.empty((n, dm.cfg.d_embed), dtype=torch.float32, device=dev) if latents else None
    zv = torch.empty((n, dm.cfg.d_device), dtype=torch.float32, device=dev) if latents else None
    z = torch.empty((n, dm.cfg.d_embed), dtype=torch.float32, device=dev) if latents else None
    lat = torch.empty(n, dtype=torch.float64, device=dev) if norm is not None else None
    bc = boxcox_struct(norm)
    if precision == "bf16":
        img = _bf16_image(dev)
        _lib.check(lib.tpcb_forward_bf16(dm.handle, params.data_ptr(), C.byref(pk.struct),
                                         devfeat.data_ptr(), n, C.byref(bc), img.data_ptr(),
                                         pred.data_ptr(), dptr(zx), dptr(zv), dptr(z), dptr(lat),
                                         status.ptr, stream_ptr()), "forward_bf16")
        return pred, zx, zv, z, lat
    if precision != "fp32":
        raise E.ValidationError(f"unknown precision {precision!r}")
    _lib.check(lib.tpcb_forward(dm.handle, params.data_ptr(), C.byref(pk.struct),
                                devfeat.data_ptr(), n, C.byref(bc), pred.data_ptr(), dptr(zx),
                                dptr(zv), dptr(z), dptr(lat), status.ptr, stream_ptr()),
               "forward")
    return pred, zx, zv, z, lat


class LargePath:
    """Layer-by-layer tensor-core forward (csrc/large.cu) for configs the
    fused kernels do not fit, e.g. full_reference_config: the transposed
    (hi, lo) weight image is built once per parameter version; the activation
    workspace grows on demand."""

    def __init__(self, dm: DeviceModel, params: torch.Tensor, with_backward: bool = False):
        self.lib = _lib.load()
        self.dm, self.params = dm, params
        self.with_backward = with_backward
        img, act = C.c_size_t(), C.c_size_t()
        _lib.check(self.lib.tpcb_large_sizes(dm.handle, 1, 1, C.byref(img), C.byref(act)),
                   "large_sizes")
        self.image = torch.zeros(img.value, dtype=torch.uint8, device=params.device)
        self.act = torch.empty(0, dtype=torch.uint8, device=params.device)
        self.prepare()

    def prepare(self) -> None:
        flags = int(self.with_backward) | (2 if getattr(self, "_table", False) else 0)
        _lib.check(self.lib.tpcb_large_prepare(self.dm.handle, self.params.data_ptr(),
                                               self.image.data_ptr(), flags, stream_ptr()),
                   "large_prepare")
        self._table = True

    @staticmethod
    def order(n_leaf: np.ndarray):
        """bucket order (the packed-index contract: stable argsort of n_leaf)
        and the token offsets in that order"""
        n_leaf = np.asarray(n_leaf, dtype=np.int64)
        perm = np.argsort(n_leaf, kind="stable").astype(np.int32)
        tok = np.zeros(len(n_leaf) + 1, dtype=np.int32)
        np.cumsum(n_leaf[perm], out=tok[1:])
        return perm, tok

    def forward(self, pk: PackedBatch, n_leaf: np.ndarray, devfeat: torch.Tensor, status: Status,
                norm=None, latents: bool = True):
        n = pk.n_ast
        perm, tok = self.order(n_leaf)
        img, act = C.c_size_t(), C.c_size_t()
        _lib.check(self.lib.tpcb_large_sizes(self.dm.handle, n, int(tok[-1]), C.byref(img),
                                             C.byref(act)), "large_sizes")
        if self.act.numel() < act.value:
            self.act = torch.empty(act.value, dtype=torch.uint8, device=self.params.device)
        dev = self.params.device
        cfg = self.dm.cfg
        pred = torch.empty(n, dtype=torch.float32, device=dev)
        zx = torch.empty((n, cfg.d_embed), dtype=torch.float32, device=dev) if latents else None
        zv = torch.empty((n, cfg.d_device), dtype=torch.float32, device=dev) if latents else None
        z = torch.empty((n, cfg.d_embed), dtype=torch.float32, device=dev) if latents else None
        lat = torch.empty(n, dtype=torch.float64, device=dev) if norm is not None else None
        bc = boxcox_struct(norm)
        _lib.check(self.lib.tpcb_large_forward(
            self.dm.handle, self.params.data_ptr(), self.image.data_ptr(), C.byref(pk.struct),
            perm.ctypes.data_as(C.c_void_p), tok.ctypes.data_as(C.c_void_p), devfeat.data_ptr(),
            n, C.byref(bc), self.act.data_ptr(), self.act.numel(), pred.data_ptr(), dptr(zx),
            dptr(zv), dptr(z), dptr(lat), status.ptr, stream_ptr()), "large_forward")
        return pred, zx, zv, z, lat


_BF16_IMG = {}


def _bf16_image(dev) -> torch.Tensor:
    """Per-device workspace for the bf16 weight image (rebuilt on every call)."""
    key = str(dev)
    if key not in _BF16_IMG:
        n = int(_lib.load().tpcb_forward_bf16_workspace())
        _BF16_IMG[key] = torch.empty(n, dtype=torch.uint8, device=dev)
    return _BF16_IMG[key]


def positional_encoding_device(ordering: np.ndarray, theta: float) -> np.ndarray:
    _need_cuda()
    lib = _lib.load()
    den = pe_denominators(theta)
    o = torch.from_numpy(np.ascontiguousarray(ordering, dtype=np.int32)).cuda()
    out = torch.empty((o.numel(), 24), dtype=torch.float64, device="cuda")
    _lib.check(lib.tpcb_positional_encoding(o.data_ptr(), o.numel(),
                                            den.ctypes.data_as(C.c_void_p), out.data_ptr(),
                                            stream_ptr()), "positional_encoding")
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# training
# ---------------------------------------------------------------------------

LOSS_MODES = {"hybrid": 0, "mse": 1, "mape": 2}
OPT_KINDS = {None: 0, "adam": 1, "sgd": 2}


class DeviceSamples:
    """A dataset resident on the device: K1-packed rows + per-sample data
    (tpcb_samples).  Built once per training run / backward call."""

    def __init__(self, rag: RaggedHost, n_leaf_max: int, status: Status, y=None, R: int = 64,
                 device="cuda", theta: float = THETA_DEFAULT):
        rows, ordering, leaf_off, devfeat = upload_ragged(rag, device)
        self.pk = pack(rows, ordering, leaf_off, rag.n_ast, n_leaf_max, rag.encoded, status, R,
                       theta)
        self.n = rag.n_ast
        self.n_leaf_host = np.asarray(rag.n_leaf, dtype=np.int64)
        self.n_leaf = torch.from_numpy(self.n_leaf_host.astype(np.int32)).to(device)
        self.devfeat = devfeat
        self.y = None
        if y is not None:
            self.y = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).to(device)
        s = _lib.Samples()
        s.x, s.ast_row = self.pk.x.data_ptr(), self.pk.ast_row.data_ptr()
        s.n_leaf, s.devfeat = self.n_leaf.data_ptr(), devfeat.data_ptr()
        s.y = self.y.data_ptr() if self.y is not None else None
        self.struct = s

    def set_targets(self, y):
        self.y = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).to(self.devfeat.device)
        self.struct.y = self.y.data_ptr()


class TrainWorkspace:
    """max_rows: samples this rank handles per step (gradient slots);
    z_rows: rows of the global [zs; zt] CMD matrix (≥ max_rows)."""

    def __init__(self, dm: DeviceModel, max_rows: int, device="cuda", z_rows: int = 0,
                 l_cap: int = 0, overlap: bool = True, wgrad_tc: bool = False):
        lib = _lib.load()
        ns, stride, zf, tf, sw = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        af = C.c_int64()
        self.l_cap = int(l_cap) if l_cap else dm.cfg.n_leaf_max
        _lib.check(lib.tpcb_train_ws_sizes(dm.handle, max_rows, self.l_cap, C.byref(ns),
                                           C.byref(stride), C.byref(zf), C.byref(tf),
                                           C.byref(sw), C.byref(af)),
                   "train_ws_sizes")
        zf = C.c_int64(max(zf.value, z_rows * dm.cfg.d_embed))
        self.max_rows = max_rows
        # zero-filled once: alignment padding between tensors is never written
        self.partial = torch.zeros(ns.value * stride.value, dtype=torch.float32, device=device)
        self.touched = torch.zeros(ns.value, dtype=torch.int32, device=device)
        self.zall = torch.empty(max(zf.value, 1), dtype=torch.float32, device=device)
        self.terms = torch.zeros(max(tf.value, 2), dtype=torch.float64, device=device)
        self.scalars = torch.zeros(8, dtype=torch.float64, device=device)
        self.step_scratch = torch.zeros(4, dtype=torch.int32, device=device)
        w = _lib.TrainWs()
        w.partial, w.slot_stride, w.n_slots = self.partial.data_ptr(), stride.value, ns.value
        w.touched, w.zall = self.touched.data_ptr(), self.zall.data_ptr()
        w.terms, w.scalars = self.terms.data_ptr(), self.scalars.data_ptr()
        w.zall_floats = self.zall.numel()
        w.l_cap = self.l_cap
        # stage counters of the overlapped reduce (owned by this workspace;
        # None = the step's reduction runs after the training kernel)
        self.stage_flags = (torch.zeros(sw.value, dtype=torch.int64, device=device)
                            if overlap else None)
        w.stage_flags = self.stage_flags.data_ptr() if overlap else None
        w.stage_flag_words = sw.value if overlap else 0
        # operand rows of the tensor-core weight-gradient GEMMs (desk shapes;
        # opt-in: measured slower than the fused per-sample gradients at bs 64,
        # DESIGN.md §5b)
        self.act = (torch.empty(af.value, dtype=torch.float32, device=device)
                    if wgrad_tc and af.value > 0 else None)
        w.act = self.act.data_ptr() if self.act is not None else None
        w.act_floats = self.act.numel() if self.act is not None else 0
        self.struct = w


def loss_struct(mode="hybrid", lambda_hybrid=1e-3, offset=0.0, alpha_cmd=0.0, cmd_order=5,
                mape_space="transformed", normalizer=None) -> _lib.LossCfg:
    c = _lib.LossCfg()
    c.mode = LOSS_MODES[mode]
    c.original_space = 1 if mape_space == "original" else 0
    c.lambda_hybrid, c.offset, c.alpha_cmd = float(lambda_hybrid), float(offset), float(alpha_cmd)
    c.cmd_order = int(cmd_order)
    c.norm = boxcox_struct(normalizer)
    return c


def optim_struct(kind, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0) -> _lib.OptimCfg:
    o = _lib.OptimCfg()
    o.kind = OPT_KINDS[kind]
    o.beta1, o.beta2, o.eps, o.weight_decay = beta1, beta2, eps, float(weight_decay)
    return o


def transpose_params(dm: DeviceModel, params: torch.Tensor, params_t: torch.Tensor) -> None:
    _lib.check(_lib.load().tpcb_transpose_params(dm.handle, params.data_ptr(),
                                                 params_t.data_ptr(), stream_ptr()), "transpose")


def run_backward(dm: DeviceModel, params: torch.Tensor, params_t: torch.Tensor,
                 src: DeviceSamples, tgt: DeviceSamples | None, loss: _lib.LossCfg,
                 ws: TrainWorkspace, status: Status):
    """One costmodel.backward over all of src (and tgt when CMD is on).
    Returns device (grad [P], pred [n_src]); loss/CMD values in ws.scalars."""
    lib = _lib.load()
    n_src = src.n
    n_tgt = tgt.n if tgt is not None else 0
    dev = params.device
    batch = torch.cat([torch.arange(n_src, dtype=torch.int32, device=dev),
                       torch.arange(n_tgt, dtype=torch.int32, device=dev)])
    grad = torch.empty(dm.n_params, dtype=torch.float32, device=dev)
    pred = torch.empty(n_src, dtype=torch.float32, device=dev)
    ws.step_scratch = torch.zeros(8, dtype=torch.int32, device=dev)
    need = max(int(src.n_leaf_host.max()), int(tgt.n_leaf_host.max()) if tgt is not None else 1)
    if need > ws.l_cap:
        raise E.ValidationError("workspace sized for fewer leaves than the batch holds")
    _lib.check(lib.tpcb_loss_backward(dm.handle, params.data_ptr(), params_t.data_ptr(),
                                      C.byref(src.struct),
                                      C.byref(tgt.struct) if tgt is not None else None,
                                      batch.data_ptr(), n_src, n_tgt, C.byref(loss),
                                      C.byref(ws.struct), ws.step_scratch.data_ptr(),
                                      grad.data_ptr(), pred.data_ptr(), status.ptr,
                                      stream_ptr()), "loss_backward")
    return grad, pred


def optimizer_step(dm: DeviceModel | None, params, params_t, grad, m, v, opt: _lib.OptimCfg,
                   lr: float, t: int) -> None:
    """nn.Adam/Sgd step on the device; dm=None steps a bare flat vector."""
    _lib.check(_lib.load().tpcb_optimizer_step(dm.handle if dm is not None else None,
                                               params.numel(), params.data_ptr(), dptr(params_t),
                                               grad.data_ptr(), dptr(m), dptr(v), C.byref(opt),
                                               float(lr), int(t), stream_ptr()), "optimizer")


class Comm:
    """NCCL communicator (tpcb_comm) bootstrapped over an initialised
    torch.distributed process group: rank 0's unique id is broadcast with
    broadcast_object_list, then every rank joins."""

    def __init__(self, rank: int, world: int, uid: bytes | None = None):
        lib = _lib.load()
        self.rank, self.world = rank, world
        if uid is None:
            import torch.distributed as dist
            buf = C.create_string_buffer(128)
            obj = [None]
            if rank == 0:
                _lib.check(lib.tpcb_nccl_unique_id(buf, 128), "nccl_unique_id")
                obj = [bytes(buf.raw)]
            if world > 1:
                dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        self._uid = C.create_string_buffer(uid, 128)
        h = C.c_void_p()
        _lib.check(lib.tpcb_nccl_comm_create(self._uid, world, rank, C.byref(h)), "nccl_comm")
        self.handle = h

    @classmethod
    def single(cls) -> "Comm":
        lib = _lib.load()
        buf = C.create_string_buffer(128)
        _lib.check(lib.tpcb_nccl_unique_id(buf, 128), "nccl_unique_id")
        return cls(0, 1, bytes(buf.raw))

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().tpcb_nccl_comm_destroy(self.handle)
            self.handle = None
