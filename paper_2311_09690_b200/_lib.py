"""ctypes binding of libtpcb200.so (the C ABI declared in include/tpcb200.h).

The library is loaded from the package directory (built in-tree by
`python -m paper_2311_09690_b200.build`).  There is deliberately no fallback:
if the library is missing every GPU entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import errors as E

LIB_PATH = Path(os.environ.get("TPCB_LIB_PATH") or
                Path(__file__).resolve().parent / "libtpcb200.so")  # (env: A/B experiments)

MAX_LAYERS, MAX_LEAF, MAX_DEC = 16, 16, 8
FEAT, FEAT_PAD, DEV_FEAT = 24, 24, 6

vp = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
sz = C.c_size_t


class Config(C.Structure):
    _fields_ = [("d_model", i32), ("n_layers", i32), ("n_heads", i32), ("d_ff", i32),
                ("d_embed", i32), ("d_device", i32), ("n_dec", i32), ("dec", i32 * MAX_DEC),
                ("n_leaf_max", i32)]


class Packed(C.Structure):
    _fields_ = [("rows_per_tile", i32), ("n_tiles_max", i32), ("x", vp), ("row_ast", vp),
                ("tile_L", vp), ("tile_first", vp), ("tile_count", vp), ("perm", vp),
                ("ast_row", vp), ("bucket_off", vp), ("n_tiles", vp)]


class BoxCox(C.Structure):
    _fields_ = [("lambda_bc", f64), ("shift", f64), ("t_mean", f64), ("t_std", f64),
                ("enabled", i32)]


class LossCfg(C.Structure):
    """tpcb_loss (hybrid / mse / mape, transformed / original space)."""
    _fields_ = [("mode", i32), ("original_space", i32), ("lambda_hybrid", f64),
                ("offset", f64), ("alpha_cmd", f64), ("cmd_order", i32),
                ("norm", BoxCox)]


class OptimCfg(C.Structure):
    _fields_ = [("kind", i32), ("beta1", f64), ("beta2", f64), ("eps", f64),
                ("weight_decay", f64)]


class Samples(C.Structure):
    _fields_ = [("x", vp), ("ast_row", vp), ("n_leaf", vp), ("devfeat", vp), ("y", vp)]


class TrainWs(C.Structure):
    _fields_ = [("partial", vp), ("slot_stride", i64), ("n_slots", i32), ("touched", vp),
                ("zall", vp), ("terms", vp), ("scalars", vp), ("zall_floats", i64),
                ("l_cap", i32), ("stage_flags", vp), ("stage_flag_words", i64),
                ("act", vp), ("act_floats", i64)]


class LargeBatch(C.Structure):
    """tpcb_large_batch (a CMD target batch of the large path)."""
    _fields_ = [("x", vp), ("ast_row", vp), ("devfeat", vp), ("h_idx", vp), ("h_tok_off", vp),
                ("h_pos", vp), ("n", i64)]


class Plan(C.Structure):
    _fields_ = [("d_batch", vp), ("d_steps", vp), ("n_steps", i32)]


# name -> (restype, argtypes)
SIGNATURES = {
    "tpcb_model_create": (i32, [C.POINTER(Config), C.POINTER(vp)]),
    "tpcb_model_destroy": (None, [vp]),
    "tpcb_model_param_count": (i64, [vp]),
    "tpcb_model_tensor_count": (i32, [vp]),
    "tpcb_model_tensor_info": (i32, [vp, i32, C.c_char_p, i32, C.POINTER(i64),
                                     C.POINTER(i32), C.POINTER(i32)]),
    "tpcb_status_string": (C.c_char_p, [i32]),
    "tpcb_last_error": (C.c_char_p, []),
    "tpcb_pack_sizes": (i32, [i64, i64, i32, i32, C.POINTER(i32), C.POINTER(sz)]),
    "tpcb_featurize_pack": (i32, [vp, i32, vp, vp, i64, i64, i32, vp, vp, sz,
                                  C.POINTER(Packed), vp, vp]),
    "tpcb_positional_encoding": (i32, [vp, i64, vp, vp, vp]),
    "tpcb_build_compact": (i32, [vp, vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp]),
    "tpcb_forward_fits": (i32, [vp, i32]),
    "tpcb_forward_rows": (i32, [vp]),
    "tpcb_large_sizes": (i32, [vp, i64, i64, C.POINTER(sz), C.POINTER(sz)]),
    "tpcb_large_prepare": (i32, [vp, vp, vp, i32, vp]),
    "tpcb_large_forward": (i32, [vp, vp, vp, C.POINTER(Packed), vp, vp, vp, i64,
                                 C.POINTER(BoxCox), vp, sz, vp, vp, vp, vp, vp, vp, vp]),
    "tpcb_large_train_ws": (i32, [vp, i64, i64, i64, i64, C.POINTER(sz)]),
    "tpcb_large_loss_backward": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64,
                                       C.POINTER(LossCfg), f64, vp, C.POINTER(LargeBatch), vp,
                                       sz, vp, vp, vp, vp, vp]),
    "tpcb_gemm3_ws": (sz, [i64, i32, i32]),
    "tpcb_gemm3": (i32, [vp, vp, i64, i32, i32, vp, i32, vp, sz, vp]),
    "tpcb_gemm3_presplit": (i32, [vp, vp, vp, vp, i64, i32, i32, vp, i32, vp]),
    "tpcb_forward": (i32, [vp, vp, C.POINTER(Packed), vp, i64, C.POINTER(BoxCox), vp, vp, vp,
                           vp, vp, vp, vp]),
    "tpcb_forward_bf16_workspace": (C.c_size_t, []),
    "tpcb_forward_bf16": (i32, [vp, vp, C.POINTER(Packed), vp, i64, C.POINTER(BoxCox), vp, vp, vp,
                                vp, vp, vp, vp, vp]),
    "tpcb_metrics": (i32, [vp, vp, i64, vp, vp]),
    "tpcb_cmd": (i32, [vp, i32, i64, i64, i32, i32, vp, vp, vp]),
    "tpcb_cmd_grid_ws": (sz, [i64, i64, i32, i32]),
    "tpcb_cmd_grid": (i32, [vp, i32, i64, i64, i32, i32, vp, vp, vp, sz, vp]),
    "tpcb_train_ws_sizes": (i32, [vp, i32, i32, C.POINTER(i32), C.POINTER(i64),
                                  C.POINTER(i64), C.POINTER(i64), C.POINTER(i64),
                                  C.POINTER(i64)]),
    "tpcb_transpose_params": (i32, [vp, vp, vp, vp]),
    "tpcb_loss_backward": (i32, [vp, vp, vp, C.POINTER(Samples), C.POINTER(Samples), vp, i32,
                                 i32, C.POINTER(LossCfg), C.POINTER(TrainWs), vp, vp, vp, vp,
                                 vp]),
    "tpcb_optimizer_step": (i32, [vp, i64, vp, vp, vp, vp, vp, C.POINTER(OptimCfg), f64, i64,
                                  vp]),
    "tpcb_optimizer_step_f64": (i32, [i64, vp, vp, vp, vp, C.POINTER(OptimCfg), f64, f64, f64,
                                      vp]),
    "tpcb_train_epoch": (i32, [vp, vp, vp, vp, vp, C.POINTER(Samples), C.POINTER(Samples),
                               C.POINTER(Plan), C.POINTER(LossCfg), C.POINTER(OptimCfg), vp, vp,
                               C.POINTER(TrainWs), vp, vp, vp, vp, vp, vp, vp, vp]),
    "tpcb_nccl_unique_id": (i32, [vp, i32]),
    "tpcb_nccl_comm_create": (i32, [vp, i32, i32, C.POINTER(vp)]),
    "tpcb_nccl_comm_destroy": (None, [vp]),
    "tpcb_nccl_allreduce_sum": (i32, [vp, vp, i64, i32, vp]),
    "tpcb_graph_create": (i32, [C.POINTER(vp)]),
    "tpcb_probe_ffma": (i32, [vp, C.POINTER(f64), vp]),
    "tpcb_debug_train_trace": (i32, [vp]),
    "tpcb_kmeans_ws_size": (i32, [i64, i32, i32, C.POINTER(sz)]),
    "tpcb_kmeanspp_init": (i32, [vp, i64, i32, i64, vp, vp, vp, vp, sz, vp]),
    "tpcb_kmeanspp_step": (i32, [vp, i64, i32, i32, f64, i64, vp, vp, vp, vp, vp, sz, vp]),
    "tpcb_kmeanspp_steps": (i32, [vp, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp]),
    "tpcb_kmeans_assign": (i32, [vp, i64, i32, vp, i32, vp, vp, vp, vp]),
    "tpcb_kmeans_assign_tc_ws": (C.c_size_t, [i32]),
    "tpcb_kmeans_assign_tc": (i32, [vp, i64, i32, vp, i32, vp, vp, vp, vp, C.c_size_t, vp]),
    "tpcb_kmeanspp_closest": (i32, [vp, i64, i32, vp, i32, vp, vp, vp, C.c_size_t, vp]),
    "tpcb_kmeanspp_cdf": (i32, [vp, i64, vp, vp, vp, C.c_size_t, vp]),
    "tpcb_kmeanspp_search": (i32, [i64, C.c_double, C.c_double, C.c_double, vp, vp, C.c_size_t,
                                   vp]),
    "tpcb_kmeans_partial": (i32, [vp, i64, i32, i32, vp, vp, vp, vp, C.c_size_t, vp]),
    "tpcb_kmeans_update": (i32, [vp, i64, i32, i32, vp, vp, vp, vp, sz, vp]),
    "tpcb_kmeans_changed": (i32, [vp, vp, i64, vp, vp]),
    "tpcb_distance_table": (i32, [vp, vp, i32, i32, vp, i32, vp, vp]),
    "tpcb_flush_l2": (i32, [vp, sz, vp]),
    "tpcb_graph_destroy": (None, [vp]),
}

STATUS_EXC = {
    1: E.ValidationError, 2: E.LeafCountExceeded, 3: E.EmptyBatch, 4: E.EmptySet,
    5: E.DimensionMismatch, 6: E.TooFewPoints, 7: E.TooFewTasks, 8: E.DomainError,
    9: E.NotFitted, 10: E.NonFiniteLoss, 11: E.UnsupportedConfig, 12: E.CudaError,
}

_lib = None


def load(path: Path | str | None = None) -> C.CDLL:
    """Load (once) and type every exported symbol; raises if anything is
    missing — there is no CPU fallback."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise E.CudaError(
            f"native library {p} not built — run `python -m paper_2311_09690_b200.build`")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError == missing export
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(status: int, what: str = "", epoch: int = -1) -> None:
    if status == 0:
        return
    exc = STATUS_EXC.get(int(status), E.TpcostError)
    lib = load()
    msg = f"{what}: {lib.tpcb_status_string(int(status)).decode()}"
    if exc is E.CudaError:
        msg += f" ({lib.tpcb_last_error().decode()})"
    if exc is E.NonFiniteLoss:
        raise E.NonFiniteLoss(epoch)
    raise exc(msg)
