"""GPU parity: K1 featurize/pack and the fused forward vs the oracle and the
reference golden vectors.  Tolerances (fp32 FFMA path, fp64 decode):
packed indices bit-exact; PE'd rows ≤ 4e-6 abs; model-space predictions
≤ 2e-5·(1+|pred|); decoded latency ≤ 1e-3 relative (north_star bar)."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import featurize as of
from oracle import predictor as op

pytestmark = pytest.mark.gpu


def _pb():
    import paper_2311_09690_b200 as pb
    return pb


def _dims(cfg):
    return op.Dims(cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.d_embed,
                   cfg.d_device, tuple(cfg.decoder_dims), cfg.n_leaf_max)


def _cfg(gm):
    pb = _pb()
    return pb.CostModelConfig(**gm.cfg)


def _c1_batch(dtype=np.float64):
    pb = _pb()
    c1 = load_golden("c1_4096")
    synth = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    n = len(c1["n_leaf"])
    return c1, pb.CompactBatch(c1["vectors"].astype(dtype), c1["ordering"].astype(np.int32),
                               c1["n_leaf"].astype(np.int64), np.zeros(n, np.int32), [synth])


@pytest.mark.parametrize("R", [32, 64, 128])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_featurize_pack_contract(R, dtype):
    from paper_2311_09690_b200 import engine
    c1, batch = _c1_batch(dtype)
    rag = batch.ragged()
    rows, ordering, leaf_off, _ = engine.upload_ragged(rag)
    st = engine.Status(rows.device)
    pk = engine.pack(rows, ordering, leaf_off, rag.n_ast, 16, False, st, R)
    st.check("pack")
    off = np.concatenate([[0], np.cumsum(c1["n_leaf"])])
    by_ast = [of.encode_rows(c1["vectors"][off[i]:off[i + 1]], c1["ordering"][off[i]:off[i + 1]])
              for i in range(len(c1["n_leaf"]))]
    want = of.pack_tiles(by_ast, 16, R)
    nt = int(pk.n_tiles.item())
    assert nt == len(want["tile_L"])
    assert np.array_equal(pk.perm.cpu().numpy(), want["perm"])
    assert np.array_equal(pk.perm.cpu().numpy(), c1["perm"])  # reference grouping order
    assert np.array_equal(pk.bucket_off.cpu().numpy(), want["bucket_offsets"])
    for k in ("tile_L", "tile_first", "tile_count"):
        assert np.array_equal(getattr(pk, k)[:nt].cpu().numpy(), want[k]), k
    assert np.array_equal(pk.ast_row.cpu().numpy(), want["ast_row"])
    row_ast = pk.row_ast[:nt * R].cpu().numpy().reshape(nt, R)
    assert np.array_equal(row_ast, want["row_ast"])
    x = pk.x[:nt * R * 24].cpu().numpy().reshape(nt, R, 24).astype(np.float64)
    assert np.all(want["tiles"][..., 24:] == 0.0)  # the oracle's pad columns (no longer stored)
    err = np.abs(x - want["tiles"][..., :24])
    assert err.max() <= 4e-6, err.max()
    assert np.all(x[want["row_mask"] == 0] == 0.0)


def test_positional_encoding_matches_reference():
    pb = _pb()
    g = load_golden("features")
    comp = pb.CompactAst(np.zeros((len(g["positions"]), 24)), tuple(g["positions"].tolist()),
                         tuple(range(9001)), len(g["positions"]))
    pe = pb.positional_encoding(comp)
    assert np.abs(pe - g["pe"]).max() <= 1e-12
    assert np.abs(pb.positional_encoding(comp, 100.0) - g["pe_theta100"]).max() <= 1e-12
    assert np.array_equal(pe[0], np.tile([0.0, 1.0], 12))


@pytest.mark.parametrize("name", ["tiny", "grad", "mid"])
def test_forward_small_configs_vs_reference(golden_model, name):
    pb = _pb()
    gm = golden_model(name)
    cfg = _cfg(gm)
    params = pb.CostModelParams(cfg, gm.T)
    rows, dev = gm.rows("in")
    inputs = [pb.EncodedInput(r, d) for r, d in zip(rows, dev)]
    pred, lat = pb.forward(params, inputs)
    tol = lambda w: 2e-5 * (1.0 + np.abs(w))  # noqa: E731
    assert np.all(np.abs(pred - gm.z["pred"]) <= tol(gm.z["pred"]))
    for k, got in (("z_x", lat.z_x), ("z_v", lat.z_v), ("z", lat.z)):
        assert np.all(np.abs(got - gm.z[k]) <= tol(gm.z[k])), k


def test_forward_desk_c1_decoded_latency_parity(golden_model):
    """C1: 4096 synthetic ASTs, trained desk checkpoint, raw compact input
    (K1 adds the PE) → decoded latency within 1e-3 relative."""
    pb = _pb()
    gm = golden_model("desk")
    cfg = _cfg(gm)
    params = pb.CostModelParams(cfg, gm.T)
    lam, shift, tm, ts, off = gm.z["norm"]
    norm = pb.BoxCoxNormalizer(lam, shift, True, tm, ts, off)
    c1, batch = _c1_batch(np.float32)
    p = pb.Predictor(params)
    pred, zx, zv, z, latency = p.forward_batch(batch, norm, latents=True)
    rel = np.abs(latency - gm.z["latency4k"]) / gm.z["latency4k"]
    assert rel.max() <= 1e-3, rel.max()
    assert np.abs(pred - gm.z["pred4k"]).max() <= 1e-3
    assert np.abs(z - gm.z["z4k"]).max() <= 1e-3


def test_predict_batch_and_predict_match_reference(golden_model):
    pb = _pb()
    gm = golden_model("desk")
    params = pb.CostModelParams(_cfg(gm), gm.T)
    lam, shift, tm, ts, off = gm.z["norm"]
    norm = pb.BoxCoxNormalizer(lam, shift, True, tm, ts, off)
    c1 = load_golden("c1_4096")
    noff = np.concatenate([[0], np.cumsum(c1["n_leaf"])])
    synth = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    dv = pb.device_vector(synth)
    idx = np.arange(0, 4096, 37)
    inputs = [pb.EncodedInput(of.encode_rows(c1["vectors"][noff[i]:noff[i + 1]],
                                             c1["ordering"][noff[i]:noff[i + 1]]), dv)
              for i in idx]
    lat = pb.predict_batch(params, inputs, norm)
    want = gm.z["latency4k"][idx]
    assert np.max(np.abs(lat - want) / want) <= 1e-3
    i = int(idx[5])
    comp = pb.CompactAst(c1["vectors"][noff[i]:noff[i + 1]],
                         tuple(c1["ordering"][noff[i]:noff[i + 1]].tolist()), (), int(c1["n_leaf"][i]))
    one = pb.predict(params, comp, synth, norm)
    assert abs(one - want[5]) / want[5] <= 1e-3


def test_forward_batch_equivariance_exact(golden_model, rng):
    """Permuting the batch permutes the outputs bit-exactly (test_costmodel.py:73-80):
    each AST's arithmetic is independent of its tile-mates."""
    pb = _pb()
    gm = golden_model("mid")
    params = pb.CostModelParams(_cfg(gm), gm.T)
    rows, dev = gm.rows("in")
    inputs = [pb.EncodedInput(r, d) for r, d in zip(rows, dev)] * 5
    pred, lat = pb.forward(params, inputs)
    perm = rng.permutation(len(inputs))
    pred_p, lat_p = pb.forward(params, [inputs[i] for i in perm])
    assert np.array_equal(pred_p, pred[perm])
    assert np.array_equal(lat_p.z, lat.z[perm])


def test_forward_zero_decoder_and_routing(golden_model, rng):
    pb = _pb()
    gm = golden_model("tiny")
    cfg = _cfg(gm)
    T = {k: v.copy() for k, v in gm.T.items()}
    T["dec.out.W"][:] = 0.0
    T["dec.out.b"][:] = 0.0
    rows, dev = gm.rows("in")
    inputs = [pb.EncodedInput(r, d) for r, d in zip(rows, dev)]
    pred, _ = pb.forward(pb.CostModelParams(cfg, T), inputs)
    assert np.array_equal(pred, np.zeros(len(inputs)))
    two = [e for e in inputs if e.n_leaf == 2][:1]
    three = [e for e in inputs if e.n_leaf == 3][:1]
    T2 = {k: v.copy() for k, v in gm.T.items()}
    base, _ = pb.forward(pb.CostModelParams(cfg, T2), two + three)
    T2["leaf_embed.3.b"] += 0.25
    bumped, _ = pb.forward(pb.CostModelParams(cfg, T2), two + three)
    assert bumped[0] == base[0] and bumped[1] != base[1]


def test_forward_errors(golden_model):
    pb = _pb()
    from paper_2311_09690_b200.errors import EmptyBatch, LeafCountExceeded
    gm = golden_model("tiny")
    params = pb.CostModelParams(_cfg(gm), gm.T)
    with pytest.raises(EmptyBatch):
        pb.forward(params, [])
    with pytest.raises(LeafCountExceeded):
        pb.forward(params, [pb.EncodedInput(np.zeros((4, 24)), np.zeros(6))])


def test_forward_large_random_vs_oracle():
    """Bigger batch, every leaf count 1..16, desk config at init."""
    pb = _pb()
    cfg = pb.desk_config(seed=3)
    params = pb.init_params(cfg)
    rng = np.random.default_rng(5)
    inputs = [pb.EncodedInput(rng.normal(size=(int(L), 24)) * 3, rng.normal(size=6))
              for L in rng.integers(1, 17, size=700)]
    pred, lat = pb.forward(params, inputs)
    want, wzx, _, wz, _ = op.forward(params.tensors, _dims(cfg), [e.matrix for e in inputs],
                                     np.stack([e.device_vector for e in inputs]))
    assert np.all(np.abs(pred - want) <= 2e-5 * (1 + np.abs(want)))
    assert np.all(np.abs(lat.z - wz) <= 2e-5 * (1 + np.abs(wz)))


@pytest.mark.parametrize("R", [128, 64])
def test_forward_desk_every_leaf_count_both_kernels(R):
    """The desk fp32 kernel (forward_f32.cu, 128-row tiles; leaf_embed staged in
    groups of 8 leaf positions, so L = 9..16 takes the multi-group path) and
    the generic kernel (64-row tiles) against the float64 oracle on every leaf
    count 1..16; same 2e-5·(1+|ref|) bar as the reference-config tests."""
    pb = _pb()
    cfg = pb.desk_config(seed=0)
    params = pb.init_params(cfg)
    rng = np.random.default_rng(11)
    n_leaf = np.concatenate([np.full(int(rng.integers(30, 200)), L) for L in range(1, 17)])
    rng.shuffle(n_leaf)
    n = len(n_leaf)
    vec = rng.uniform(0.0, 8.0, size=(int(n_leaf.sum()), 24))
    ordering = np.concatenate([rng.permutation(28)[:L] for L in n_leaf]).astype(np.int32)
    synth = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    batch = pb.CompactBatch(vec, ordering, n_leaf.astype(np.int64), np.zeros(n, np.int32), [synth])
    p = pb.Predictor(params, rows_per_tile=R)
    assert p.R == R
    pred, zx, zv, z, _ = p.forward_batch(batch, latents=True)
    off = np.concatenate([[0], np.cumsum(n_leaf)])
    x = [of.encode_rows(vec[off[i]:off[i + 1]], ordering[off[i]:off[i + 1]]) for i in range(n)]
    dv = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    ref = op.forward(params.tensors, _dims(cfg), x, np.tile(dv, (n, 1)))
    tol = lambda w: 2e-5 * (1.0 + np.abs(w))  # noqa: E731
    assert np.all(np.abs(pred - ref[0]) <= tol(ref[0])), np.abs(pred - ref[0]).max()
    for got, want, k in ((zx, ref[1], "z_x"), (zv, ref[2], "z_v"), (z, ref[3], "z")):
        assert np.all(np.abs(got - want) <= tol(want)), k


def test_forward_desk_default_tiles_use_the_desk_kernel():
    pb = _pb()
    assert pb.Predictor(pb.init_params(pb.desk_config(seed=0))).R == 128
    small = pb.desk_config(seed=0, d_model=32, d_ff=64, d_embed=16)
    assert pb.Predictor(pb.init_params(small)).R == 64


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_forward_batch_pipelined_equals_one_shot(precision):
    """The chunked two-stream bulk path (H2D of chunk i+1 overlapping the
    forward of chunk i, device-side leaf offsets / device features) returns
    the one-shot results bit for bit: every kernel is per AST / token row."""
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import synth
    from paper_2311_09690_b200.dataset import fit_boxcox
    import torch
    data = synth.generate(20000, seed=9)
    norm = fit_boxcox(data.latency)
    devs = [pb.DeviceSpec("a", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0),
            pb.DeviceSpec("b", 1590.0, 16.0, 320.0, 40, 8100.0, 4.0)]
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa: E731
    batch = pb.CompactBatch(pin(data.vectors.astype(np.float32)),
                            pin(data.ordering.astype(np.int32)), pin(data.n_leaf),
                            pin((np.arange(data.n) % 2).astype(np.int32)), devs)
    params = pb.init_params(pb.desk_config(seed=4))
    p = pb.Predictor(params, precision=precision)
    one = p.forward_batch(batch, None, latents=True)  # n <= CHUNK: one shot
    p.CHUNK = 3000  # several pipelined chunks (instance attribute shadows the class default)
    many = p.forward_batch(batch, None, latents=True)
    for a, b in zip(one[:4], many[:4]):
        assert np.array_equal(a, b)
    assert one[4] is None and many[4] is None
    # a bad leaf count in a later piece: the same error and global index as
    # the one-shot path (checked per piece, after earlier pieces were queued)
    from paper_2311_09690_b200.errors import LeafCountExceeded
    nl = np.array(data.n_leaf)
    bad = 17000
    nl[bad] = 0
    bad_batch = pb.CompactBatch(batch.vectors[: int(nl.sum())], batch.ordering[: int(nl.sum())],
                                nl, batch.device_index, devs)
    with pytest.raises(LeafCountExceeded, match=f"input {bad} "):
        p.forward_batch(bad_batch, None)


def test_forward_batch_concurrent_threads_on_one_predictor():
    """Two threads running the pipelined bulk path on one Predictor (shared
    read-only params, disjoint batches — SURVEY 8(b) threading): each gets its
    own staging buffers and copy stream, so the results equal the serial ones."""
    import threading
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import synth
    import torch
    devs = [pb.DeviceSpec("a", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)]
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa: E731
    batches = []
    for seed in (21, 22):
        d = synth.generate(12000, seed=seed)
        batches.append(pb.CompactBatch(pin(d.vectors.astype(np.float32)),
                                       pin(d.ordering.astype(np.int32)), pin(d.n_leaf),
                                       np.zeros(d.n, np.int32), devs))
    p = pb.Predictor(pb.init_params(pb.desk_config(seed=6)), precision="bf16")
    p.CHUNK = 2500
    serial = [p.forward_batch(b, None)[0] for b in batches]
    out = [None, None]

    def run(i):
        for _ in range(3):
            out[i] = p.forward_batch(batches[i], None)[0]

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for a, b in zip(serial, out):
        assert np.array_equal(a, b)


def test_pack_positional_table_cache_per_theta():
    """K1 keeps one PE table per (device, θ): packs alternating between two θ
    values each match the float64 oracle rows (rounded to f32) for their own
    θ (within K1's 4e-6 row bar) — a cached table is never reused for another θ."""
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import _lib, engine, synth
    data = synth.generate(3000, seed=31)
    dv = pb.device_vector(pb.DeviceSpec("a", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0))
    rag = engine.RaggedHost(rows=data.vectors.astype(np.float32), ordering=data.ordering,
                            n_leaf=data.n_leaf, devfeat=np.tile(dv, (data.n, 1)).astype(np.float32),
                            encoded=False)
    rows, ordering, leaf_off, _ = engine.upload_ragged(rag)
    st = engine.Status(rows.device)
    off = np.concatenate([[0], np.cumsum(data.n_leaf)])
    for theta in (10000.0, 777.0, 10000.0, 777.0):
        pk = engine.pack(rows, ordering, leaf_off, data.n, 16, False, st, 128, theta)
        x = pk.x.cpu().numpy().reshape(-1, _lib.FEAT_PAD)
        ast_row = pk.ast_row.cpu().numpy()
        for i in (0, 1, 777, 2999):
            want = of.encode_rows(data.vectors[off[i]:off[i + 1]].astype(np.float32),
                                  data.ordering[off[i]:off[i + 1]], theta)
            got = x[ast_row[i]:ast_row[i] + data.n_leaf[i], :24]
            assert np.abs(got - want).max() <= 4e-6, (theta, i)  # K1's own bar (see above)
