"""GPU: training through the large-model path (csrc/large.cu,
large_training.py) — one batch's loss and full parameter gradient against
the float64 oracle's costmodel.backward restatement (desk config with a
mixed-leaf-count batch, and full_reference_config; the original-space
relative loss; the CMD term with a mixed-leaf-count target batch, the
default of full_reference_config), a few optimizer steps on the desk
config matching the fused trainer, and finetune(full_reference_config)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import featurize as of
from oracle import predictor as op

pytestmark = pytest.mark.gpu

DV = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)


def _batch(n, seed, same_leaf=None):
    c1 = load_golden("c1_4096")
    off = np.concatenate([[0], np.cumsum(c1["n_leaf"])])
    rng = np.random.default_rng(seed)
    cand = np.arange(len(c1["n_leaf"]))
    if same_leaf is not None:
        cand = cand[c1["n_leaf"] == same_leaf]
    idx = rng.permutation(cand)[:n]
    rows = [c1["vectors"][off[i]:off[i + 1]] for i in idx]
    order = [c1["ordering"][off[i]:off[i + 1]] for i in idx]
    y = rng.normal(size=n)
    return rows, order, y


def _rag(rows, order):
    from paper_2311_09690_b200 import engine
    n = len(rows)
    return engine.RaggedHost(rows=np.concatenate(rows).astype(np.float32),
                             ordering=np.concatenate(order).astype(np.int32),
                             n_leaf=np.array([len(r) for r in rows]),
                             devfeat=np.tile(DV.astype(np.float32), (n, 1)), encoded=False)


def _oracle_grad(cfg, T, rows, order, y, lam=1e-3):
    dims = op.Dims(cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.d_embed, cfg.d_device,
                   tuple(cfg.decoder_dims), cfg.n_leaf_max)
    x = [of.encode_rows(r, o) for r, o in zip(rows, order)]
    pred, _, _, _, tapes = op.forward(T, dims, x, np.tile(DV, (len(x), 1)))
    val, dpred = op.loss_and_grad(pred, y, "hybrid", lam, 0.0)
    G = op.backward_from(T, dims, tapes, dpred, None)
    return val, G


def _compare(got_loss, got, ref_loss, ref, tol):
    assert abs(got_loss - ref_loss) <= tol * max(1.0, abs(ref_loss))
    # floor: 1e-4 of the largest gradient anywhere — attn.bk's gradient is
    # analytically zero (softmax is shift-invariant per query row), so only
    # rounding noise remains there in both implementations
    floor = 1e-4 * max(np.abs(g).max() for g in ref.values())
    for name, g in ref.items():
        scale = max(np.abs(g).max(), floor)
        err = np.abs(got[name] - g).max()
        assert err <= tol * scale, (name, err, scale)


def test_desk_mixed_batch_gradient_vs_oracle():
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200.large_training import large_loss_backward
    cfg = pb.desk_config(seed=0)
    params = pb.init_params(cfg)
    rows, order, y = _batch(48, 3)
    loss, G, _ = large_loss_backward(params, _rag(rows, order), y)
    ref_loss, ref = _oracle_grad(cfg, params.tensors, rows, order, y)
    _compare(loss, G, ref_loss, ref, 2e-3)


def test_full_reference_config_gradient_vs_oracle():
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200.large_training import large_loss_backward
    cfg = pb.full_reference_config()
    params = pb.init_params(cfg)
    rows, order, y = _batch(6, 5, same_leaf=3)
    loss, G, _ = large_loss_backward(params, _rag(rows, order), y)
    ref_loss, ref = _oracle_grad(cfg, params.tensors, rows, order, y)
    _compare(loss, G, ref_loss, ref, 5e-3)


def test_desk_large_trainer_tracks_fused_trainer():
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import engine, synth
    from paper_2311_09690_b200.dataset import fit_boxcox
    from paper_2311_09690_b200.large_training import LargeTrainer
    from paper_2311_09690_b200.training import Trainer
    data = synth.generate(2048, seed=1)
    norm = fit_boxcox(data.latency)
    dv = np.tile(DV.astype(np.float32), (data.n, 1))
    rag = engine.RaggedHost(rows=data.vectors.astype(np.float32), ordering=data.ordering,
                            n_leaf=data.n_leaf, devfeat=dv, encoded=False)
    cfg = pb.desk_config(seed=0)
    loss = engine.loss_struct("hybrid", cfg.lambda_hybrid, norm.loss_offset)
    y = norm.encode(data.latency)
    T0 = pb.init_params(cfg).tensors
    big = LargeTrainer(cfg, T0, rag, y, loss)
    fused = Trainer(cfg, T0, rag, y, loss, use_graph=False)
    flat, steps = big.plan(np.random.default_rng(0))
    big.run_epoch(1e-3, flat, steps)
    fused.run_epoch(1e-3, flat, steps)
    a, b = big.tensors(), fused.tensors()
    for k in a:
        if k.endswith("attn.bk"):
            # zero gradient analytically: Adam turns each implementation's
            # fp32 rounding noise into (different) small steps
            continue
        assert np.allclose(a[k], b[k], rtol=2e-3, atol=2e-4), k


def _oracle_grad_cmd(cfg, T, rows, order, y, trows, torder, alpha, k=5, lam=1e-3):
    from oracle import moments as om
    dims = op.Dims(cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.d_embed, cfg.d_device,
                   tuple(cfg.decoder_dims), cfg.n_leaf_max)
    x = [of.encode_rows(r, o) for r, o in zip(rows, order)]
    xt = [of.encode_rows(r, o) for r, o in zip(trows, torder)]
    pred, _, _, z, tapes = op.forward(T, dims, x, np.tile(DV, (len(x), 1)))
    _, _, _, zt, tapes_t = op.forward(T, dims, xt, np.tile(DV, (len(xt), 1)))
    val, dpred = op.loss_and_grad(pred, y, "hybrid", lam, 0.0)
    c, gs, gt = om.cmd_grad(z, zt, k)
    G = op.backward_from(T, dims, tapes, dpred, alpha * gs)
    op.backward_from(T, dims, tapes_t, np.zeros(len(xt)), alpha * gt, G)
    return val + alpha * c, G, c


@pytest.mark.parametrize("name", ["desk", "full"])
def test_cmd_gradient_vs_oracle(name):
    """CMD fine-tuning step on the large path: source batch of one leaf
    count, target batch mixing leaf counts (the reference's fallback pool),
    CMD over [zs; zt] in input order — value, loss and every gradient vs the
    oracle (costmodel.py:529-570)."""
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200.large_training import large_loss_backward
    cfg = pb.desk_config(seed=0) if name == "desk" else pb.full_reference_config()
    params = pb.init_params(cfg)
    if name == "desk":
        rows, order, y = _batch(32, 7, same_leaf=4)
        trows, torder, _ = _batch(24, 8)
    else:
        # full config (11 layers x 985 ReLU units): batches whose ReLU
        # pre-activations all stay >= 4e-6 away from 0 in the float64 oracle
        # (source: the batch of test_full_reference_config_gradient_vs_oracle,
        # target: 1.4e-5).  A pre-activation within the fp32-class rounding
        # of this path (~1e-6 relative) flips its mask against float64 —
        # measured on another batch (min 3e-6 in enc8): that FFN column off
        # by 3 % in the alpha = 0 gradient too
        rows, order, y = _batch(6, 5, same_leaf=3)
        trows, torder, _ = _batch(5, 15)
    trows = [r + np.where((np.arange(24) >= 10) & (np.arange(24) < 16), 2.0, 0.0) for r in trows]
    loss, G, cmd = large_loss_backward(params, _rag(rows, order), y, alpha_cmd=1.0,
                                       target_rag=_rag(trows, torder))
    ref_loss, ref, ref_cmd = _oracle_grad_cmd(cfg, params.tensors, rows, order, y, trows,
                                              torder, 1.0)
    assert abs(cmd - ref_cmd) <= 2e-5 * ref_cmd, (cmd, ref_cmd)
    _compare(loss, G, ref_loss, ref, 2e-3 if name == "desk" else 5e-3)


def test_original_space_loss_vs_oracle():
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200.large_training import large_loss_backward
    cfg = pb.desk_config(seed=0)
    params = pb.init_params(cfg)
    rows, order, _ = _batch(40, 9)
    norm = pb.BoxCoxNormalizer(lambda_bc=-0.07, shift=0.0, fitted=True, t_mean=0.2, t_std=0.9,
                               loss_offset=1.3)
    y = np.random.default_rng(2).uniform(-1.0, 1.0, size=40)
    loss, G, _ = large_loss_backward(params, _rag(rows, order), y, lambda_hybrid=0.1,
                                     mape_space="original", normalizer=norm)
    dims = op.Dims(cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.d_embed, cfg.d_device,
                   tuple(cfg.decoder_dims), cfg.n_leaf_max)
    x = [of.encode_rows(r, o) for r, o in zip(rows, order)]
    pred, _, _, _, tapes = op.forward(params.tensors, dims, x, np.tile(DV, (len(x), 1)))
    val, dpred = op.loss_and_grad(pred, y, "hybrid", 0.1, 0.0, "original",
                                  (-0.07, 0.0, 0.2, 0.9))
    ref = op.backward_from(params.tensors, dims, tapes, dpred, None)
    _compare(loss, G, val, ref, 2e-3)


def test_finetune_full_reference_config_runs():
    """finetune() on full_reference_config (alpha_cmd = 1 by default,
    costmodel.py:89-96) routes to the large path with the CMD term: one
    short epoch, finite losses, positive CMD, deterministic."""
    import paper_2311_09690_b200 as pb
    c1 = load_golden("c1_4096")
    off = np.concatenate([[0], np.cumsum(c1["n_leaf"])])
    idx = np.arange(0, 4096, 16)  # 256 samples
    samples, splits = [], {}
    for j, i in enumerate(idx):
        comp = pb.CompactAst(c1["vectors"][off[i]:off[i + 1]],
                             tuple(c1["ordering"][off[i]:off[i + 1]].tolist()), (),
                             int(c1["n_leaf"][i]))
        smp = pb.Sample(f"s{j}", "t0", "m0", "synth0", comp, float(c1["latency"][i]))
        samples.append(smp)
        splits[smp.id] = "train" if j % 8 else "valid"
    ds = pb.Dataset(samples=samples, splits=splits)
    devices = {"synth0": pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)}
    from dataclasses import replace
    cfg = replace(pb.full_reference_config(), epochs=1, batch_size=32)
    assert cfg.alpha_cmd == 1.0
    params = pb.init_params(cfg)
    norm = pb.fit_boxcox([s.latency_s for s in ds.subset("train")])
    shift = np.where((np.arange(24) >= 10) & (np.arange(24) < 16), 2.0, 0.0)
    dv = pb.device_vector(devices["synth0"])
    tgt = [pb.EncodedInput(of.encode_rows(s.compact.leaf_vectors, s.compact.ordering) + shift, dv)
           for s in ds.subset("valid")]
    a = pb.finetune(params, ds, tgt, cfg, devices, norm)
    b = pb.finetune(params, ds, tgt, cfg, devices, norm)
    assert np.isfinite(a.log[0].train_loss) and a.log[0].cmd > 0
    assert [r.__dict__ for r in a.log] == [r.__dict__ for r in b.log]
