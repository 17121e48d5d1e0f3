"""GPU: the bf16 tensor-core forward (tcgen05, the C5 sweep mode) against the
float64 oracle and the fp32 parity path.

Stated tolerance of the bf16 mode (north_star: "bf16 path tolerance stated
separately"), on the reference-trained desk checkpoint and the reference's
4,096-AST C1 set: decoded latency within 0.10 relative of the float64
oracle for every AST and 0.02 relative on average (measured with the
current two-warpgroup kernel: max 5.1e-2, mean 1.1e-2); model-space predictions within 0.05·(1+|p|).  The fp32 mode
keeps the 1e-3 bar (test_gpu_forward.py)."""

import numpy as np
import pytest

from conftest import GoldenModel, load_golden
from oracle import featurize as of
from oracle import predictor as op

pytestmark = pytest.mark.gpu


def _setup():
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import engine
    gm = GoldenModel("desk")
    params = pb.CostModelParams(pb.CostModelConfig(**gm.cfg), gm.T)
    c1 = load_golden("c1_4096")
    lam, sh, tm, ts, loff = gm.z["norm"]
    norm = pb.BoxCoxNormalizer(lam, sh, True, tm, ts, loff)
    dv = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    n = len(c1["n_leaf"])
    rag = engine.RaggedHost(rows=c1["vectors"].astype(np.float32), ordering=c1["ordering"],
                            n_leaf=c1["n_leaf"], devfeat=np.tile(dv.astype(np.float32), (n, 1)),
                            encoded=False)
    return pb, gm, params, c1, norm, dv, rag


def test_bf16_forward_vs_oracle_and_fp32():
    pb, gm, params, c1, norm, dv, rag = _setup()
    out = {}
    for prec in ("fp32", "bf16"):
        pred, zx, zv, z, lat = pb.Predictor(params, precision=prec).forward_ragged(rag, norm)
        out[prec] = (pred.double().cpu().numpy(), lat.cpu().numpy(), zv.cpu().numpy())
    # float64 oracle on the same inputs
    off = np.concatenate([[0], np.cumsum(c1["n_leaf"])])
    x = [of.encode_rows(c1["vectors"][off[i]:off[i + 1]], c1["ordering"][off[i]:off[i + 1]])
         for i in range(len(c1["n_leaf"]))]
    dims = op.Dims(gm.cfg["d_model"], gm.cfg["n_layers"], gm.cfg["n_heads"], gm.cfg["d_ff"],
                   gm.cfg["d_embed"], gm.cfg["d_device"], tuple(gm.cfg["decoder_dims"]),
                   gm.cfg["n_leaf_max"])
    ref_pred = op.forward(gm.T, dims, x, np.tile(dv, (len(x), 1)))[0]
    ref_lat = norm.decode(ref_pred)
    pred_b, lat_b, zv_b = out["bf16"]
    assert np.all(np.abs(pred_b - ref_pred) <= 0.05 * (1 + np.abs(ref_pred)))
    rel = np.abs(lat_b - ref_lat) / np.abs(ref_lat)
    print(f"bf16 decoded-latency rel err vs fp64: max {rel.max():.3e} mean {rel.mean():.3e}")
    assert rel.max() <= 0.10, rel.max()
    assert rel.mean() <= 0.02, rel.mean()
    # the device MLP never touches the tensor cores: identical to the fp32 mode
    assert np.allclose(zv_b, out["fp32"][2], rtol=1e-6, atol=1e-6)


def test_bf16_forward_rejects_other_shapes():
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200.errors import UnsupportedConfig
    cfg = pb.desk_config(seed=0, d_model=32, d_ff=64, d_embed=16)
    p = pb.Predictor(pb.init_params(cfg), precision="bf16")
    c1 = load_golden("c1_4096")
    synth = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    batch = pb.CompactBatch(c1["vectors"][:40], c1["ordering"][:40].astype(np.int32),
                            np.array([1] * 40, np.int64), np.zeros(40, np.int32), [synth])
    with pytest.raises(UnsupportedConfig):
        p.forward_batch(batch)


def test_bf16_forward_every_leaf_count():
    """leaf_embed runs on the tensor cores with per-L staging (L ≥ 8 restages
    the B chunks in groups): every leaf count 1..16, several tiles per bucket,
    against the float64 oracle, same stated tolerance on z_x and predictions."""
    import paper_2311_09690_b200 as pb
    cfg = pb.desk_config(seed=0)
    params = pb.init_params(cfg)
    rng = np.random.default_rng(7)
    n_leaf = np.concatenate([np.full(int(rng.integers(40, 300)), L) for L in range(1, 17)])
    rng.shuffle(n_leaf)
    n = len(n_leaf)
    vec = rng.uniform(0.0, 8.0, size=(int(n_leaf.sum()), 24))
    ordering = np.concatenate([rng.permutation(28)[:L] for L in n_leaf]).astype(np.int32)
    synth = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    batch = pb.CompactBatch(vec, ordering, n_leaf.astype(np.int64), np.zeros(n, np.int32), [synth])
    pred, zx, _, _, _ = pb.Predictor(params, precision="bf16").forward_batch(batch, latents=True)
    off = np.concatenate([[0], np.cumsum(n_leaf)])
    x = [of.encode_rows(vec[off[i]:off[i + 1]], ordering[off[i]:off[i + 1]]) for i in range(n)]
    dims = op.Dims(cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.d_embed, cfg.d_device,
                   tuple(cfg.decoder_dims), cfg.n_leaf_max)
    dv = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    ref = op.forward(params.tensors, dims, x, np.tile(dv, (n, 1)))
    ref_pred, ref_zx = ref[0], ref[1]
    scale = np.abs(ref_zx).max(axis=1, keepdims=True) + 1e-3
    ezx = (np.abs(zx - ref_zx) / scale).max(axis=1)
    ep = np.abs(pred - ref_pred) / (1 + np.abs(ref_pred))
    for L in range(1, 17):
        m = n_leaf == L
        print(f"L={L:2d} n={m.sum():3d} z_x max {ezx[m].max():.3e} pred max {ep[m].max():.3e} "
              f"mean {ep[m].mean():.3e}")
    # random-init weights on uniform(0, 8) features: larger activations than the
    # trained checkpoint above, hence the looser per-AST bound
    assert ezx.max() <= 0.05
    assert ep.max() <= 0.10 and ep.mean() <= 0.02
