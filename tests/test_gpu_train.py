"""GPU parity of the training path vs the reference's own golden vectors:
backward (every LossSpec variant incl. CMD), standalone CMD, the optimizers.

Tolerances (fp32 accumulate; CMD statistics in fp64):
  gradients   per tensor  max|Δ| ≤ 2e-4 · max|ref| + 1e-6
  loss value  relative    ≤ 1e-5
  CMD (fp64 standalone)   value rel ≤ 1e-12, gradients ≤ 1e-10 abs
  Adam / SGD  (drop-in nn, float64 state) bit-exact vs the reference
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import featurize as of

pytestmark = pytest.mark.gpu

CASES = {
    "mse": dict(mode="mse"),
    "hyb": dict(mode="hybrid", lambda_hybrid=1e-3, offset=0.75),
    "mape": dict(mode="mape", offset=0.75),
    "cmd": dict(mode="hybrid", lambda_hybrid=1e-3, offset=0.75, alpha_cmd=1.0, cmd_order=5),
    "cmd3": dict(mode="hybrid", lambda_hybrid=1e-3, offset=0.75, alpha_cmd=0.5, cmd_order=3),
    "orig": dict(mode="hybrid", lambda_hybrid=0.1, mape_space="original"),
}


def _pb():
    import paper_2311_09690_b200 as pb
    return pb


def _assert_grads(got, gm, case, scale=2e-4):
    ref = gm.grads(case)
    for k, T in gm.T.items():
        want = ref.get(k, np.zeros_like(T))
        err = np.abs(got[k] - want).max()
        assert err <= scale * np.abs(want).max() + 1e-6, (k, err, np.abs(want).max())


@pytest.mark.parametrize("name", ["tiny", "grad", "mid"])
@pytest.mark.parametrize("case", list(CASES))
def test_backward_small_configs_vs_reference(golden_model, name, case):
    pb = _pb()
    from paper_2311_09690_b200.costmodel import LossSpec, backward
    gm = golden_model(name)
    params = pb.CostModelParams(pb.CostModelConfig(**gm.cfg), gm.T)
    rows, dev = gm.rows("in")
    trows, tdev = gm.rows("tg")
    batch = [pb.EncodedInput(r, d) for r, d in zip(rows, dev)]
    tb = [pb.EncodedInput(r, d) for r, d in zip(trows, tdev)]
    kw = dict(CASES[case])
    if case == "orig":
        kw["normalizer"] = pb.BoxCoxNormalizer(-0.07, 0.0, True, 0.2, 0.9, 1.3)
    val, grads, aux = backward(params, batch, gm.z["targets"], LossSpec(**kw),
                               target_batch=tb if case.startswith("cmd") else None)
    assert val == pytest.approx(float(gm.z[f"bw.{case}.loss"]), rel=1e-5)
    if case.startswith("cmd"):
        assert aux["cmd"] == pytest.approx(float(gm.z[f"bw.{case}.cmd"]), rel=1e-5)
    np.testing.assert_allclose(aux["pred"], gm.z["pred"], rtol=2e-5, atol=2e-5)
    _assert_grads(grads, gm, case)


@pytest.mark.parametrize("case,wgrad_tc", [("hyb", False), ("orig", False), ("cmd", False),
                                           ("hyb", True), ("orig", True)])
def test_backward_desk_trained_batch(golden_model, case, wgrad_tc):
    """A reference batch: 64 samples of one bucket (+64 shifted targets);
    wgrad_tc: the encoder weight gradients as tcgen05 GEMMs over the batch's
    256 token rows (csrc/wgrad.cu), same tolerance."""
    pb = _pb()
    from paper_2311_09690_b200.costmodel import LossSpec, backward
    gm = golden_model("desk")
    params = pb.CostModelParams(pb.CostModelConfig(**gm.cfg), gm.T)
    c1 = load_golden("c1_4096")
    off = np.concatenate([[0], np.cumsum(c1["n_leaf"])])
    dv = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    enc = lambda i: of.encode_rows(c1["vectors"][off[i]:off[i + 1]],  # noqa: E731
                                   c1["ordering"][off[i]:off[i + 1]])
    shift = np.where((np.arange(24) >= 10) & (np.arange(24) < 16), 2.0, 0.0)
    batch = [pb.EncodedInput(enc(i), dv) for i in gm.z["batch_idx"]]
    tb = [pb.EncodedInput(enc(i) + shift, dv) for i in gm.z["tbatch_idx"]]
    lam, sh, tm, ts, loff = gm.z["norm"]
    norm = pb.BoxCoxNormalizer(lam, sh, True, tm, ts, loff)
    spec = {"hyb": LossSpec(mode="hybrid", lambda_hybrid=1e-3, offset=loff),
            "orig": LossSpec(mode="hybrid", lambda_hybrid=0.1, mape_space="original",
                             normalizer=norm),
            "cmd": LossSpec(mode="hybrid", lambda_hybrid=1e-3, offset=loff, alpha_cmd=1.0)}[case]
    val, grads, aux = backward(params, batch, gm.z["batch_y"], spec,
                               target_batch=tb if case == "cmd" else None, wgrad_tc=wgrad_tc)
    assert val == pytest.approx(float(gm.z[f"bw.{case}.loss"]), rel=1e-5)
    _assert_grads(grads, gm, case)


def test_backward_errors(golden_model):
    pb = _pb()
    from paper_2311_09690_b200.costmodel import LossSpec, backward
    from paper_2311_09690_b200.errors import EmptyBatch, ValidationError
    gm = golden_model("tiny")
    params = pb.CostModelParams(pb.CostModelConfig(**gm.cfg), gm.T)
    rows, dev = gm.rows("in")
    batch = [pb.EncodedInput(r, d) for r, d in zip(rows, dev)]
    with pytest.raises(ValidationError):
        backward(params, batch[:3], np.ones(2), LossSpec())
    with pytest.raises(EmptyBatch):
        backward(params, [], np.ones(0), LossSpec())
    with pytest.raises(ValidationError):  # shifted labels must be positive
        backward(params, batch[:2], np.array([-2.0, 1.0]), LossSpec(offset=0.5))
    with pytest.raises(ValidationError):  # original space needs a normalizer
        backward(params, batch[:2], np.ones(2), LossSpec(mape_space="original"))


def test_cmd_standalone_fp64_vs_reference():
    pb = _pb()
    from paper_2311_09690_b200.costmodel import cmd_grad
    from paper_2311_09690_b200.errors import DimensionMismatch, EmptySet
    g = load_golden("cmd")
    for c in range(12):
        zs, zt = g[f"c{c}.zs"], g[f"c{c}.zt"]
        for k in (5, 3):
            v, gs, gt = cmd_grad(zs, zt, k)
            assert v == pytest.approx(float(g[f"c{c}.k{k}.value"]), rel=1e-12, abs=1e-14)
            np.testing.assert_allclose(gs, g[f"c{c}.k{k}.gs"], rtol=1e-9, atol=1e-10)
            np.testing.assert_allclose(gt, g[f"c{c}.k{k}.gt"], rtol=1e-9, atol=1e-10)
    assert pb.costmodel.cmd(np.array([[0.0], [1.0]]), np.array([[0.5], [0.5]])) == \
        pytest.approx(0.3125, abs=1e-12)
    s = np.random.default_rng(1).normal(size=(10, 4))
    assert pb.costmodel.cmd(s, s.copy()) == 0.0
    a, b = np.random.default_rng(2).normal(size=(9, 3)), np.random.default_rng(3).normal(size=(14, 3))
    assert pb.costmodel.cmd(a, b) == pytest.approx(pb.costmodel.cmd(b, a), rel=1e-13)
    with pytest.raises(EmptySet):
        pb.costmodel.cmd(np.empty((0, 2)), np.ones((3, 2)))
    with pytest.raises(DimensionMismatch):
        pb.costmodel.cmd(np.ones((2, 2)), np.ones((3, 3)))


def test_adam_sgd_vs_reference():
    from paper_2311_09690_b200 import nn
    g = load_golden("adam")
    names = [k[3:] for k in g.files if k.startswith("p0.")]
    params = {n: g["p0." + n].copy() for n in names}
    opt = nn.Adam(names, weight_decay=0.01)
    for step in range(3):
        grads = {n: g[f"g{step}." + n] for n in names}
        opt.step(params, grads, 1e-2)
        for n in names:  # float64 state, the reference's operation order: bit-exact
            assert params[n].dtype == np.float64
            np.testing.assert_array_equal(params[n], g[f"p{step + 1}." + n], err_msg=n)
    sgd = nn.Sgd(names, weight_decay=0.1)
    params = {n: g["p3." + n].copy() for n in names}
    sgd.step(params, {n: g["g2." + n] for n in names}, 0.5)
    for n in names:
        np.testing.assert_array_equal(params[n], g["sgd." + n], err_msg=n)
    with pytest.raises(ValueError):  # a changed parameter set is rejected, not mis-scattered
        bad = dict(params)
        bad[names[0]] = np.zeros((3, 3))
        sgd.step(bad, {n: g["g2." + n] for n in names}, 0.5)


def test_cmd_grid_kernels_vs_oracle_large_sets():
    """cmd_between-sized sets take the multi-block kernels (tpcb_cmd_grid):
    value and gradient vs the float64 oracle (itself pinned to the reference,
    tests/test_oracle_golden.py), cmd(S, S) exactly 0, f32 input, ties in
    the extrema routed to the first row."""
    from oracle import moments as om
    from paper_2311_09690_b200.costmodel import CMD_GRID_ROWS, cmd, cmd_grad
    rng = np.random.default_rng(7)
    ns, nt = 20000, 13001
    assert ns + nt >= CMD_GRID_ROWS
    zs = rng.normal(size=(ns, 32))
    zt = rng.normal(0.2, 1.3, size=(nt, 32))
    zs[5, 3] = zs[17, 3] = 9.0   # tie on the max: first row (5) carries the support grad
    zt[100, 7] = -9.0
    # k 3 / 4 / 5: compile-time orders of pass AC; 2 and 7: the runtime-order
    # pass AC; de 24: the generic (shared-memory coefficient) pass E
    for k, de in ((5, 32), (3, 32), (2, 32), (7, 32), (5, 24), (4, 24)):
        v, gs, gt = cmd_grad(zs[:, :de], zt[:, :de], k)
        wv, wgs, wgt = om.cmd_grad(zs[:, :de], zt[:, :de], k)
        assert v == pytest.approx(wv, rel=1e-11), (k, de)
        np.testing.assert_allclose(gs, wgs, rtol=1e-7, atol=1e-13)
        np.testing.assert_allclose(gt, wgt, rtol=1e-7, atol=1e-13)
    big = rng.normal(size=(CMD_GRID_ROWS, 32))
    assert cmd(big, big.copy()) == 0.0
    v32 = cmd(zs.astype(np.float32), zt.astype(np.float32))
    w32 = om.cmd_grad(zs.astype(np.float32).astype(np.float64),
                      zt.astype(np.float32).astype(np.float64), 5)[0]
    assert v32 == pytest.approx(w32, rel=1e-11)
