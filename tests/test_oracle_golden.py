"""Pin the CPU oracle to the reference: golden vectors + the reference test
suite's own known answers.  CPU only (no GPU, no /root/reference needed)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import featurize as of
from oracle import lloyd, moments, optim
from oracle import predictor as op


def dims(cfg):
    return op.Dims(cfg["d_model"], cfg["n_layers"], cfg["n_heads"], cfg["d_ff"],
                   cfg["d_embed"], cfg["d_device"], cfg["decoder_dims"], cfg["n_leaf_max"])


def ragged_rows(z, prefix=""):
    n_leaf = z[prefix + "n_leaf"]
    off = np.concatenate([[0], np.cumsum(n_leaf)])
    return n_leaf, off


# ---------------------------------------------------------------- features

def test_pe_known_answers():
    g = load_golden("features")
    pe = of.positional_rows(g["positions"])
    assert np.array_equal(pe, g["pe"])  # same float64 formula: bit-exact
    assert np.array_equal(of.positional_rows(g["positions"], 100.0), g["pe_theta100"])
    assert np.array_equal(pe[0], np.tile([0.0, 1.0], 12))  # test_features.py:139-143
    assert np.all(np.abs(pe) <= 1.0)


def test_device_vector_known_answers():
    g = load_golden("features")
    v = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    assert np.array_equal(v, g["dev_synth"])
    v4 = of.device_features(1590, 16, 320, 40, 8100, 4)
    assert np.array_equal(v4, g["dev_t4"])


def test_encode_and_bucket_perm_synth512():
    g = load_golden("synth512")
    n_leaf, off = ragged_rows(g)
    rows = np.concatenate([of.encode_rows(g["vectors"][off[i]:off[i + 1]],
                                          g["ordering"][off[i]:off[i + 1]])
                           for i in range(len(n_leaf))])
    assert np.array_equal(rows, g["enc_rows"])
    perm, boff = of.bucket_perm(n_leaf, 16)
    assert np.array_equal(perm, g["perm"])  # bit-exact packed index contract
    assert np.array_equal(perm, np.argsort(n_leaf, kind="stable"))
    assert boff[-1] == len(n_leaf)


def test_pack_tiles_contract():
    g = load_golden("synth512")
    n_leaf, off = ragged_rows(g)
    by_ast = [g["enc_rows"][off[i]:off[i + 1]] for i in range(len(n_leaf))]
    pk = of.pack_tiles(by_ast, 16, 128)
    # every AST appears exactly once, with its own rows, bucket-contiguous
    assert np.array_equal(np.sort(pk["perm"]), np.arange(len(n_leaf)))
    flat = pk["tiles"].reshape(-1, 32)
    for i in range(len(n_leaf)):
        r = pk["ast_row"][i]
        assert np.array_equal(flat[r:r + n_leaf[i], :24], by_ast[i])
    assert pk["row_mask"].sum() == n_leaf.sum()
    assert np.all(pk["tiles"][pk["row_mask"] == 0] == 0.0)
    assert np.all(pk["tile_count"] * pk["tile_L"] <= 128)


# ----------------------------------------------------------- forward/backward

@pytest.mark.parametrize("name", ["tiny", "grad", "mid"])
def test_forward_small_configs(golden_model, name):
    gm = golden_model(name)
    dm = dims(gm.cfg)
    rows, dev = gm.rows("in")
    pred, zx, zv, z, _ = op.forward(gm.T, dm, rows, dev)
    np.testing.assert_allclose(pred, gm.z["pred"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(zx, gm.z["z_x"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(zv, gm.z["z_v"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(z, gm.z["z"], rtol=1e-12, atol=1e-13)


def _oracle_backward(gm, case, spec):
    dm = dims(gm.cfg)
    rows, dev = gm.rows("in")
    y = gm.z["targets"]
    pred, zx, zv, z, tapes = op.forward(gm.T, dm, rows, dev)
    val, dpred = op.loss_and_grad(pred, y, **spec.get("loss", {}))
    dzs = None
    G = {}
    if "cmd" in spec:
        alpha, k = spec["cmd"]
        trows, tdev = gm.rows("tg")
        _, _, _, zt, ttapes = op.forward(gm.T, dm, trows, tdev)
        cv, gs, gt = moments.cmd_grad(z, zt, k)
        val += alpha * cv
        dzs = alpha * gs
        op.backward_from(gm.T, dm, tapes, dpred, dzs, G)
        op.backward_from(gm.T, dm, ttapes, np.zeros(len(trows)), alpha * gt, G)
    else:
        op.backward_from(gm.T, dm, tapes, dpred, None, G)
    return val, G


SPECS = {
    "mse": {"loss": dict(mode="mse")},
    "hyb": {"loss": dict(mode="hybrid", lam_h=1e-3, offset=0.75)},
    "mape": {"loss": dict(mode="mape", offset=0.75)},
    "cmd": {"loss": dict(mode="hybrid", lam_h=1e-3, offset=0.75), "cmd": (1.0, 5)},
    "cmd3": {"loss": dict(mode="hybrid", lam_h=1e-3, offset=0.75), "cmd": (0.5, 3)},
    "orig": {"loss": dict(mode="hybrid", lam_h=0.1, space="original",
                          norm=(-0.07, 0.0, 0.2, 0.9))},
}


@pytest.mark.parametrize("name", ["tiny", "grad", "mid"])
@pytest.mark.parametrize("case", list(SPECS))
def test_backward_small_configs(golden_model, name, case):
    gm = golden_model(name)
    val, G = _oracle_backward(gm, case, SPECS[case])
    assert val == pytest.approx(float(gm.z[f"bw.{case}.loss"]), rel=1e-11)
    ref = gm.grads(case)
    for k in gm.T:
        want = ref.get(k, np.zeros_like(gm.T[k]))
        got = G.get(k, np.zeros_like(gm.T[k]))
        np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-12, err_msg=k)


def test_desk_trained_forward_and_decode(golden_model):
    gm = golden_model("desk")
    c1 = load_golden("c1_4096")
    dm = dims(gm.cfg)
    n_leaf, off = ragged_rows(c1)
    rows = [of.encode_rows(c1["vectors"][off[i]:off[i + 1]], c1["ordering"][off[i]:off[i + 1]])
            for i in range(len(n_leaf))]
    dev = np.tile(of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0), (len(rows), 1))
    pred, zx, zv, z, _ = op.forward(gm.T, dm, rows, dev)
    np.testing.assert_allclose(pred, gm.z["pred4k"], rtol=1e-10, atol=1e-11)
    np.testing.assert_allclose(z, gm.z["z4k"], rtol=1e-10, atol=1e-11)
    lam, shift, tm, ts, _ = gm.z["norm"]
    lat = op.boxcox_decode(pred, lam, shift, tm, ts)
    np.testing.assert_allclose(lat, gm.z["latency4k"], rtol=1e-9)


def test_desk_trained_backward(golden_model):
    gm = golden_model("desk")
    c1 = load_golden("c1_4096")
    dm = dims(gm.cfg)
    n_leaf, off = ragged_rows(c1)
    enc = lambda i: of.encode_rows(c1["vectors"][off[i]:off[i + 1]],  # noqa: E731
                                   c1["ordering"][off[i]:off[i + 1]])
    dv = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    shift = np.where((np.arange(24) >= 10) & (np.arange(24) < 16), 2.0, 0.0)
    rows = [enc(i) for i in gm.z["batch_idx"]]
    trows = [enc(i) + shift for i in gm.z["tbatch_idx"]]
    dev = np.tile(dv, (len(rows), 1))
    lam, sh, tm, ts, loff = gm.z["norm"]
    y = gm.z["batch_y"]
    for case, spec in (("hyb", dict(mode="hybrid", lam_h=1e-3, offset=loff)),
                       ("orig", dict(mode="hybrid", lam_h=0.1, space="original",
                                     norm=(lam, sh, tm, ts))),
                       ("cmd", dict(mode="hybrid", lam_h=1e-3, offset=loff))):
        pred, _, _, z, tapes = op.forward(gm.T, dm, rows, dev)
        val, dpred = op.loss_and_grad(pred, y, **spec)
        G = {}
        if case == "cmd":
            _, _, _, zt, tt = op.forward(gm.T, dm, trows, np.tile(dv, (len(trows), 1)))
            cv, gs, gt = moments.cmd_grad(z, zt, 5)
            val += cv
            op.backward_from(gm.T, dm, tapes, dpred, gs, G)
            op.backward_from(gm.T, dm, tt, np.zeros(len(trows)), gt, G)
        else:
            op.backward_from(gm.T, dm, tapes, dpred, None, G)
        assert val == pytest.approx(float(gm.z[f"bw.{case}.loss"]), rel=1e-10)
        ref = gm.grads(case)
        for k in gm.T:
            want = ref.get(k, np.zeros_like(gm.T[k]))
            got = G.get(k, np.zeros_like(gm.T[k]))
            np.testing.assert_allclose(got, want, rtol=1e-8, atol=1e-12, err_msg=k)


# ---------------------------------------------------------------------- CMD

def test_cmd_golden():
    g = load_golden("cmd")
    for c in range(12):
        zs, zt = g[f"c{c}.zs"], g[f"c{c}.zt"]
        for k in (5, 3):
            v, gs, gt = moments.cmd_grad(zs, zt, k)
            assert v == pytest.approx(float(g[f"c{c}.k{k}.value"]), rel=1e-12, abs=1e-14)
            np.testing.assert_allclose(gs, g[f"c{c}.k{k}.gs"], rtol=1e-10, atol=1e-13)
            np.testing.assert_allclose(gt, g[f"c{c}.k{k}.gt"], rtol=1e-10, atol=1e-13)
    # reference hand value (test_costmodel.py:128-131)
    assert moments.cmd_grad(np.array([[0.0], [1.0]]), np.array([[0.5], [0.5]]))[0] == \
        pytest.approx(0.3125, abs=1e-12)
    assert float(g["hand"]) == pytest.approx(0.3125, abs=1e-12)
    s = np.random.default_rng(1).normal(size=(10, 4))
    assert moments.cmd_grad(s, s.copy())[0] == 0.0


def test_losses_known_answers():
    v, _ = op.loss_and_grad(np.array([2.0]), np.array([1.0]), offset=0.0)
    assert v == pytest.approx(1.001)  # test_costmodel.py:115-120


# --------------------------------------------------------------------- Adam

def test_adam_sgd_golden():
    g = load_golden("adam")
    names = [k[3:] for k in g.files if k.startswith("p0.")]
    p = np.concatenate([g["p0." + n].ravel() for n in names])
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    for step in range(3):
        gr = np.concatenate([g[f"g{step}." + n].ravel() for n in names])
        optim.adam_step(p, gr, m, v, step + 1, 1e-2, wd=0.01)
        want = np.concatenate([g[f"p{step + 1}." + n].ravel() for n in names])
        assert np.array_equal(p, want)
    optim.sgd_step(p, gr, 0.5, wd=0.1)
    assert np.array_equal(p, np.concatenate([g["sgd." + n].ravel() for n in names]))


# -------------------------------------------------------------------- kmeans

def test_kmeans_hand_runs():
    g = load_golden("kmeans")
    c, a, s, _ = lloyd.kmeans(np.array([0.0, 0.1, 5.0, 10.0, 10.1]), 2,
                              init_centers=np.array([0.05, 10.05]))
    assert np.array_equal(c, g["five_centers"]) and np.array_equal(a, g["five_assign"])
    assert c[0, 0] == pytest.approx(1.7, abs=1e-12)  # test_sampling.py:39-44
    assert a.tolist() == [0, 0, 0, 1, 1]
    c, a, s, _ = lloyd.kmeans(np.array([[0.0], [0.0], [0.0], [9.0]]), 2,
                              init_centers=np.array([[0.0], [0.0]]))
    assert np.array_equal(a, g["rep_assign"]) and np.array_equal(c, g["rep_centers"])


def test_kmeans_golden_bit_exact():
    g = load_golden("kmeans")
    x = g["cli_x"]
    rows = g["cli_task_rows"]
    off = np.concatenate([[0], np.cumsum(rows)])
    feats = [x[off[i]:off[i + 1]] for i in range(len(rows))]
    for kappa, seed in ((4, 0), (9, 3)):
        init = lloyd.kmeanspp(x, kappa, np.random.default_rng(seed))
        assert np.array_equal(init, g[f"k{kappa}.init"])
        c, a, s, _ = lloyd.kmeans(x, kappa, seed=seed)
        assert np.array_equal(c, g[f"k{kappa}.centers"])
        assert np.array_equal(a, g[f"k{kappa}.assign"])
        psi = lloyd.psi_table(c, feats)
        assert np.array_equal(psi, g[f"k{kappa}.psi"])
        picked = lloyd.greedy_pick(psi, s)
        ids = [str(t) for t in g["cli_task_ids"]]
        assert [ids[i] for i in picked] == [str(t) for t in g[f"k{kappa}.selected"]]
    xb = g["blob_x"]
    assert np.array_equal(lloyd.kmeanspp(xb, 16, np.random.default_rng(11)), g["blob_init"])
    c, a, s, _ = lloyd.kmeans(xb, 16, seed=11)
    assert np.array_equal(c, g["blob_centers"]) and np.array_equal(a, g["blob_assign"])


def test_select_tasks_hand_example():
    # test_sampling.py:143-146 — [A, B]
    x = np.array([0.0, 0.1, 5.0, 10.0, 10.1])
    feats = [np.array([[0.0], [0.1]]), np.array([[10.0], [10.1]]), np.array([[5.0]])]
    c, a, s, _ = lloyd.kmeans(x, 2, init_centers=np.array([0.05, 10.05]))
    psi = lloyd.psi_table(c, feats)
    assert psi[0, 0] == pytest.approx(1.65, abs=1e-12)
    assert psi[1, 1] == pytest.approx(0.05, abs=1e-12)
    assert lloyd.greedy_pick(psi, s) == [0, 1]
