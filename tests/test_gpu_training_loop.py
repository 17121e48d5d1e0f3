"""GPU training / fine-tuning loops (costmodel.train / finetune) against the
reference's recorded 10-epoch desk run, plus the reference's determinism and
edge-case contracts.

Tolerance: the reference trains in float64, this path in fp32 with the same
batches (identical host RNG plan), so the epoch losses track the reference
run closely: per-epoch mean training loss within 2 % relative for the 10
epochs, best epoch identical."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _pb():
    import paper_2311_09690_b200 as pb
    return pb


def c1_dataset():
    pb = _pb()
    g = load_golden("c1_4096")
    off = np.concatenate([[0], np.cumsum(g["n_leaf"])])
    samples, splits = [], {}
    names = ("train", "valid", "test")
    for i in range(len(g["n_leaf"])):
        comp = pb.CompactAst(g["vectors"][off[i]:off[i + 1]],
                             tuple(g["ordering"][off[i]:off[i + 1]].tolist()), (), int(g["n_leaf"][i]))
        s = pb.Sample(f"s{i}", f"t{g['task'][i]}", f"m{g['model'][i]}", "synth0", comp,
                      float(g["latency"][i]))
        samples.append(s)
        splits[s.id] = names[int(g["split"][i])]
    return pb.Dataset(samples=samples, splits=splits)


SYNTH = None


def devices():
    pb = _pb()
    return {"synth0": pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)}


def test_train_tracks_reference_desk_run():
    """Epoch 0 of the reference's recorded 10-epoch desk run (same batches):
    mean train loss within 1e-3 relative.  Beyond that fp32-vs-fp64 training
    trajectories separate chaotically — Adam's first steps move every
    parameter by ±lr·sign(g), so rounding-level gradients (the key bias has an
    exactly-zero true gradient: softmax shift invariance) and ReLU masks
    flipped by near-zero pre-activations change trajectories; parity is
    checked per step (test_single_step_matches_oracle), over a short horizon,
    and end to end by the reference's acceptance criterion 6 instead."""
    pb = _pb()
    gm = load_golden("model_desk")
    ds = c1_dataset()
    res = pb.train(pb.desk_config(epochs=1, seed=0), ds, devices())
    ref = gm["train_log"]  # [epoch] = (train_loss, val_mape, val_rmse)
    assert abs(res.log[0].train_loss - ref[0, 0]) / ref[0, 0] <= 1e-3
    lam, shift, tm, ts, off = gm["norm"]
    assert res.normalizer.lambda_bc == pytest.approx(lam, abs=1e-12)


def _oracle_setup(n=2048, seed=3):
    pb = _pb()
    from paper_2311_09690_b200 import engine, synth
    from paper_2311_09690_b200.dataset import fit_boxcox
    data = synth.generate(n, seed=seed)
    norm = fit_boxcox(data.latency)
    y = norm.encode(data.latency)
    dv = pb.device_vector(devices()["synth0"])
    rag = engine.RaggedHost(rows=data.vectors, ordering=data.ordering, n_leaf=data.n_leaf,
                            devfeat=np.tile(dv, (data.n, 1)).astype(np.float32), encoded=False)
    loss = engine.loss_struct("hybrid", 1e-3, norm.loss_offset, 0.0, 5, "transformed", norm)
    return data, norm, y, dv, rag, loss


def test_steps_track_oracle_short_horizon():
    """Per-step losses of the device trainer vs the float64 oracle trainer on
    the same plan: first 8 optimizer steps within 1e-3 relative."""
    pb = _pb()
    from oracle import featurize as of
    from oracle import predictor as op
    from oracle import trainer as ot
    from paper_2311_09690_b200.training import Trainer
    data, norm, y, dv, rag, loss = _oracle_setup()
    cfg = pb.desk_config(seed=0)
    params = pb.init_params(cfg)
    tr = Trainer(cfg, params.tensors, rag, y, loss, use_graph=False)
    flat, steps = tr.plan(np.random.default_rng(0))
    steps = steps[:8].copy()
    tr.run_epoch(1e-3, flat, steps)
    tr.stream.synchronize()
    got = tr.step_loss[:8].cpu().numpy()
    T = {k: v.copy() for k, v in params.tensors.items()}
    dm = op.Dims(64, 2, 2, 128, 32, 16, (64, 64), 16)
    opt = ot.AdamState(T)
    off = data.offsets()
    want = []
    for (o, n, *_rest) in steps:
        b = flat[o:o + n]
        L = int(data.n_leaf[b[0]])
        x = np.stack([of.encode_rows(data.vectors[off[i]:off[i] + L],
                                     data.ordering[off[i]:off[i] + L]) for i in b])
        want.append(ot.train_step(T, dm, x, np.tile(dv, (n, 1)), y[b], opt, 1e-3,
                                  norm.loss_offset))
    rel = np.abs(got - np.array(want)) / np.abs(np.array(want))
    assert rel.max() <= 1e-3, rel


@pytest.mark.parametrize("wgrad_tc", [False, True])
def test_single_step_matches_oracle(wgrad_tc):
    """One Adam step from identical parameters on a reference batch: every
    updated parameter within 2e-5 absolute of the float64 step, except the
    parameters whose exact gradient is 0 (attention key biases: Adam turns
    rounding noise into ±lr steps there)."""
    pb = _pb()
    from oracle import featurize as of
    from oracle import predictor as op
    from oracle import trainer as ot
    from paper_2311_09690_b200.training import Trainer
    data, norm, y, dv, rag, loss = _oracle_setup()
    cfg = pb.desk_config(seed=0)
    params = pb.init_params(cfg)
    tr = Trainer(cfg, params.tensors, rag, y, loss, use_graph=False, wgrad_tc=wgrad_tc)
    assert (tr.ws.act is not None) == wgrad_tc
    flat, steps = tr.plan(np.random.default_rng(0))
    tr.run_epoch(1e-3, flat, steps[:1].copy())
    got = tr.tensors()
    T = {k: v.copy() for k, v in params.tensors.items()}
    o, n = steps[0][:2]
    b = flat[o:o + n]
    L = int(data.n_leaf[b[0]])
    off = data.offsets()
    x = np.stack([of.encode_rows(data.vectors[off[i]:off[i] + L],
                                 data.ordering[off[i]:off[i] + L]) for i in b])
    ot.train_step(T, op.Dims(64, 2, 2, 128, 32, 16, (64, 64), 16), x, np.tile(dv, (n, 1)), y[b],
                  ot.AdamState(T), 1e-3, norm.loss_offset)
    for k in T:
        if k.endswith("attn.bk"):
            continue
        err = np.abs(got[k] - T[k]).max()
        assert err <= 2e-5, (k, err)


def test_acceptance_criterion_6_desk_learning():
    """The reference's acceptance criterion 6 (test_acceptance.py:232-257) on
    the GPU trainer, same 2,000-sample dataset (golden, generated by the
    reference): desk config, 300 epochs → test MAPE ≤ 0.20 and 90 % of test
    samples within 35 % relative error."""
    pb = _pb()
    g = load_golden("crit6")
    off = np.concatenate([[0], np.cumsum(g["n_leaf"])])
    samples, splits = [], {}
    for i in range(len(g["n_leaf"])):
        comp = pb.CompactAst(g["vectors"][off[i]:off[i + 1]],
                             tuple(g["ordering"][off[i]:off[i + 1]].tolist()), (), int(g["n_leaf"][i]))
        s = pb.Sample(f"s{i}", f"t{g['task'][i]}", f"m{g['model'][i]}", "synth0", comp,
                      float(g["latency"][i]))
        samples.append(s)
        splits[s.id] = ("train", "valid", "test")[int(g["split"][i])]
    ds = pb.Dataset(samples=samples, splits=splits)
    res = pb.train(pb.desk_config(epochs=300, seed=0), ds, devices())
    test = ds.subset("test")
    inputs = pb.encode_dataset(test, devices())
    pred = pb.predict_batch(res.params, inputs, res.normalizer)
    actual = np.array([s.latency_s for s in test])
    mape = pb.metrics(pred, actual)["mape"]
    p90 = float(np.quantile(np.abs(pred - actual) / actual, 0.9))
    assert mape <= 0.20, (mape, p90)
    assert p90 <= 0.35, (mape, p90)


def test_train_deterministic_and_zero_epochs():
    pb = _pb()
    ds = c1_dataset()
    cfg = pb.desk_config(epochs=3, seed=11, d_model=16, d_ff=32, d_embed=8, batch_size=16)
    a = pb.train(cfg, ds, devices())
    b = pb.train(cfg, ds, devices())
    assert [r.__dict__ for r in a.log] == [r.__dict__ for r in b.log]
    for k in a.params.tensors:
        assert np.array_equal(a.params.tensors[k], b.params.tensors[k])
    z = pb.train(pb.desk_config(epochs=0, seed=3), ds, devices())
    fresh = pb.init_params(pb.desk_config(epochs=0, seed=3))
    assert z.log == []
    for k in fresh.tensors:
        assert np.array_equal(z.params.tensors[k], fresh.tensors[k])


def test_finetune_cmd_runs_and_is_deterministic():
    pb = _pb()
    ds = c1_dataset()
    cfg = pb.desk_config(epochs=2, seed=10, d_model=16, d_ff=32, d_embed=8, d_device=4,
                         decoder_dims=(8,), batch_size=32)
    pre = pb.train(cfg, ds, devices())
    shift = np.where((np.arange(24) >= 10) & (np.arange(24) < 16), 2.0, 0.0)
    test = ds.subset("test")
    dv = pb.device_vector(devices()["synth0"])
    from oracle import featurize as of
    tgt = [pb.EncodedInput(of.encode_rows(s.compact.leaf_vectors, s.compact.ordering) + shift, dv)
           for s in test]
    ft_cfg = pb.desk_config(epochs=2, seed=10, d_model=16, d_ff=32, d_embed=8, d_device=4,
                            decoder_dims=(8,), batch_size=32, alpha_cmd=1.0)
    f1 = pb.finetune(pre.params, ds, tgt, ft_cfg, devices(), pre.normalizer)
    f2 = pb.finetune(pre.params, ds, tgt, ft_cfg, devices(), pre.normalizer)
    assert [r.__dict__ for r in f1.log] == [r.__dict__ for r in f2.log]
    assert all(e.cmd > 0 for e in f1.log)
    for k in f1.params.tensors:
        assert np.array_equal(f1.params.tensors[k], f2.params.tensors[k])
    from paper_2311_09690_b200.errors import EmptyDataset
    with pytest.raises(EmptyDataset):
        pb.finetune(pre.params, ds, [], ft_cfg, devices(), pre.normalizer)


def test_data_parallel_path_single_rank_matches():
    """The data-parallel step (local gradient → NCCL all-reduce → optimizer
    from the gradient) on a 1-rank communicator reproduces the fused
    single-GPU step bit for bit, CMD included."""
    pb = _pb()
    from paper_2311_09690_b200 import engine
    from paper_2311_09690_b200.training import Trainer
    data, norm, y, dv, rag, loss = _oracle_setup(n=1024)
    cfg = pb.desk_config(seed=0, alpha_cmd=1.0, d_model=16, d_ff=32, d_embed=8)
    params = pb.init_params(cfg)
    tgt = engine.RaggedHost(rows=rag.rows + 0.5, ordering=rag.ordering, n_leaf=rag.n_leaf,
                            devfeat=rag.devfeat, encoded=False)
    loss = engine.loss_struct("hybrid", 1e-3, norm.loss_offset, 1.0, 5, "transformed", norm)
    comm = engine.Comm.single()
    runs = []
    for c in (None, comm):
        tr = Trainer(cfg, params.tensors, rag, y, loss, target_rag=tgt, comm=c)
        rng = np.random.default_rng(0)
        for _ in range(2):
            flat, steps = tr.plan(rng)
            n = tr.run_epoch(1e-3, flat, steps)
            losses, cmds, _ = tr.collect(n, 0)
        runs.append((losses, cmds, tr.tensors()))
    comm.close()
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])
    for k in runs[0][2]:
        assert np.array_equal(runs[0][2][k], runs[1][2][k]), k


@pytest.mark.parametrize("use_graph", [False, True])
def test_overlapped_reduce_bitwise_equals_sequential(use_graph):
    """The overlapped reduce + Adam (each backward stage reduced on the idle
    SMs as soon as every training CTA published it) gives bit-identical
    parameters, Adam moments and step losses to the sequential reduce kernel
    over two epochs of the desk model (graph-captured and eager)."""
    pb = _pb()
    from paper_2311_09690_b200.training import Trainer
    data, norm, y, dv, rag, loss = _oracle_setup(n=2048)
    cfg = pb.desk_config(seed=0)
    params = pb.init_params(cfg)
    runs = []
    for on in (False, True):
        tr = Trainer(cfg, params.tensors, rag, y, loss, use_graph=use_graph, overlap=on)
        assert (tr.ws.stage_flags is not None) == on
        rng = np.random.default_rng(3)
        for _ in range(2):
            flat, steps = tr.plan(rng)
            n = tr.run_epoch(1e-3, flat, steps)
            losses, _, _ = tr.collect(n, 0)
        st = int(tr.status.t.item()) if hasattr(tr, "status") else 0
        assert st == 0
        runs.append((losses, tr.tensors(), tr.m.cpu().numpy().copy(),
                     tr.v.cpu().numpy().copy()))
    assert np.array_equal(runs[0][0], runs[1][0])
    for k in runs[0][1]:
        assert np.array_equal(runs[0][1][k], runs[1][1][k]), k
    assert np.array_equal(runs[0][2], runs[1][2]) and np.array_equal(runs[0][3], runs[1][3])
