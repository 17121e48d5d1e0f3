"""GPU: the layer-by-layer tensor-core path (csrc/large.cu) — the 3xTF32
tcgen05 GEMM against an fp64 matmul, and the full_reference_config forward
(d 716, 11 layers, 46.7 M parameters) against the float64
oracle: model-space predictions within 1e-3·(1+|p|) and latents within
1e-3 relative to their scale (the fp32-accumulate parity bar).  The desk
config forced through the same path must agree with the fused kernel."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import featurize as of
from oracle import predictor as op

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (300, 985, 716), (517, 69, 24), (1000, 2148, 736),
                                   (128, 256, 4096)])
def test_gemm3_vs_fp64(M, N, K):
    from paper_2311_09690_b200 import _lib
    lib = _lib.load()
    g = torch.Generator().manual_seed(M + N + K)
    a = torch.randn(M, K, generator=g, dtype=torch.float32)
    b = torch.randn(N, K, generator=g, dtype=torch.float32)
    ref = (a.double() @ b.double().T).numpy()
    ad, bd = a.cuda(), b.cuda()
    ldc = (N + 31) // 32 * 32
    c = torch.full((M, ldc), float("nan"), device="cuda")
    ws = torch.empty(int(lib.tpcb_gemm3_ws(M, N, K)), dtype=torch.uint8, device="cuda")
    _lib.check(lib.tpcb_gemm3(ad.data_ptr(), bd.data_ptr(), M, N, K, c.data_ptr(), ldc,
                              ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream),
               "gemm3")
    out = c.cpu().numpy()
    # |a·b| ~ sqrt(K) for unit normals.  Single-pass TF32 would err by
    # ~2^-11·sqrt(K) (≈ 0.03 max at K = 716); 3xTF32 is fp32-class, bounded by
    # the tensor core's fp32 accumulation (measured max ≈ 3e-5·sqrt(K))
    err = np.abs(out[:, :N] - ref).max()
    print(f"gemm3 {M}x{N}x{K}: max abs err {err:.3e}")
    assert err <= 8e-5 * np.sqrt(K)
    assert np.all(out[:, N:] == 0)


def _inputs(n, seed=0):
    c1 = load_golden("c1_4096")
    off = np.concatenate([[0], np.cumsum(c1["n_leaf"])])
    idx = np.random.default_rng(seed).permutation(len(c1["n_leaf"]))[:n]
    rows = [c1["vectors"][off[i]:off[i + 1]] for i in idx]
    order = [c1["ordering"][off[i]:off[i + 1]] for i in idx]
    return rows, order


def _run(cfg, tensors, rows, order, path="auto"):
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import engine
    params = pb.CostModelParams(cfg, tensors)
    p = pb.Predictor(params, path=path)
    dv = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0).astype(np.float32)
    n = len(rows)
    rag = engine.RaggedHost(rows=np.concatenate(rows).astype(np.float32),
                            ordering=np.concatenate(order).astype(np.int32),
                            n_leaf=np.array([len(r) for r in rows]),
                            devfeat=np.tile(dv, (n, 1)), encoded=False)
    pred, zx, zv, z, _ = p.forward_ragged(rag)
    return p, [t.double().cpu().numpy() for t in (pred, zx, zv, z)]


def _oracle(cfg, tensors, rows, order):
    x = [of.encode_rows(r, o) for r, o in zip(rows, order)]
    dims = op.Dims(cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.d_embed, cfg.d_device,
                   tuple(cfg.decoder_dims), cfg.n_leaf_max)
    dv = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    return op.forward(tensors, dims, x, np.tile(dv, (len(x), 1)))[:4]


def test_full_reference_config_forward_vs_oracle():
    import paper_2311_09690_b200 as pb
    cfg = pb.full_reference_config()
    tensors = pb.init_params(cfg).tensors
    rows, order = _inputs(96)
    p, got = _run(cfg, tensors, rows, order)
    assert p.large is not None  # the fused kernels cannot hold d = 716
    ref = _oracle(cfg, tensors, rows, order)
    assert np.all(np.abs(got[0] - ref[0]) <= 1e-3 * (1 + np.abs(ref[0]))), \
        np.abs(got[0] - ref[0]).max()
    for g, r in zip(got[1:], ref[1:]):
        assert np.abs(g - r).max() <= 1e-3 * max(1.0, np.abs(r).max())


def test_desk_config_large_path_matches_fused_and_oracle():
    import paper_2311_09690_b200 as pb
    cfg = pb.desk_config(seed=0)
    tensors = pb.init_params(cfg).tensors
    rows, order = _inputs(300, seed=1)
    _, big = _run(cfg, tensors, rows, order, path="large")
    _, fused = _run(cfg, tensors, rows, order, path="fused")
    ref = _oracle(cfg, tensors, rows, order)
    for g, f, r in zip(big, fused, ref):
        tol = 1e-4 * max(1.0, np.abs(r).max())
        assert np.abs(g - r).max() <= tol
        assert np.abs(g - f).max() <= tol
