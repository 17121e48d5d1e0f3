"""C-ABI library checks that need no GPU: the in-tree libtpcb200.so loads,
exports every function include/tpcb200.h declares, and the host-only model
handle reproduces the reference's canonical tensor layout."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT
from oracle import predictor as op

HEADER = ROOT / "include" / "tpcb200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tpcb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2311_09690_b200 import _lib
    if not _lib.LIB_PATH.exists():
        from paper_2311_09690_b200 import build
        build.build()
    return _lib.load()


def test_header_declares_functions():
    names = declared_functions()
    assert "tpcb_forward" in names and "tpcb_featurize_pack" in names
    assert len(names) >= 10


def test_every_declared_symbol_exported_and_typed(lib):
    from paper_2311_09690_b200 import _lib
    for name in declared_functions():
        assert hasattr(lib, name), f"{name} not exported"
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"


def test_status_strings(lib):
    assert lib.tpcb_status_string(0) == b"ok"
    assert lib.tpcb_status_string(2) == b"LeafCountExceeded"
    assert lib.tpcb_status_string(8) == b"DomainError"


@pytest.mark.parametrize("cfg", [
    dict(d_model=64, n_layers=2, n_heads=2, d_ff=128, d_embed=32, d_device=16,
         decoder_dims=(64, 64), n_leaf_max=16),
    dict(d_model=8, n_layers=1, n_heads=2, d_ff=8, d_embed=6, d_device=3,
         decoder_dims=(6,), n_leaf_max=3),
])
def test_model_layout_matches_reference_order(lib, cfg):
    from paper_2311_09690_b200 import _lib
    c = _lib.Config()
    for k in ("d_model", "n_layers", "n_heads", "d_ff", "d_embed", "d_device", "n_leaf_max"):
        setattr(c, k, cfg[k])
    c.n_dec = len(cfg["decoder_dims"])
    for i, w in enumerate(cfg["decoder_dims"]):
        c.dec[i] = w
    h = C.c_void_p()
    assert lib.tpcb_model_create(C.byref(c), C.byref(h)) == 0
    specs = op.tensor_specs(op.Dims(**cfg))
    assert lib.tpcb_model_tensor_count(h) == len(specs)
    buf = C.create_string_buffer(128)
    off, r, cc = C.c_int64(), C.c_int32(), C.c_int32()
    expect_off = 0
    n_real = 0
    for i, (name, shape) in enumerate(specs):
        assert lib.tpcb_model_tensor_info(h, i, buf, 128, C.byref(off), C.byref(r),
                                          C.byref(cc)) == 0
        assert buf.value.decode() == name
        got = (r.value, cc.value) if cc.value else (r.value,)
        assert got == shape
        expect_off = (expect_off + 3) // 4 * 4  # 16-byte aligned tensors, creation order
        assert off.value == expect_off
        expect_off += int(np.prod(shape))
        n_real += int(np.prod(shape))
    assert lib.tpcb_model_param_count(h) == (expect_off + 3) // 4 * 4
    if cfg["d_model"] == 64:
        assert n_real == 354_577
    lib.tpcb_model_destroy(h)


def test_model_create_rejects_bad_config(lib):
    from paper_2311_09690_b200 import _lib
    c = _lib.Config()
    c.d_model, c.n_layers, c.n_heads, c.d_ff, c.d_embed, c.d_device = 10, 1, 3, 8, 4, 4
    c.n_dec, c.n_leaf_max = 0, 4
    h = C.c_void_p()
    assert lib.tpcb_model_create(C.byref(c), C.byref(h)) == 1  # ValidationError
    c.n_heads, c.n_leaf_max = 2, 17
    assert lib.tpcb_model_create(C.byref(c), C.byref(h)) == 11  # beyond kernel limits


def test_pack_sizes(lib):
    ntm, ws = C.c_int32(), C.c_size_t()
    assert lib.tpcb_pack_sizes(4096, 14912, 16, 64, C.byref(ntm), C.byref(ws)) == 0
    assert ntm.value >= 14912 // 64
    assert lib.tpcb_pack_sizes(10, 10, 16, 8, C.byref(ntm), C.byref(ws)) == 11
