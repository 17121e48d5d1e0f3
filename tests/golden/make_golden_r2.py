"""Round-2 golden fixtures, produced by running the REFERENCE (`tpcost`):

    python tests/golden/make_golden_r2.py

* finetune.npz — one reference `finetune` run (costmodel.py:721-780) on the
  acceptance-criterion-7 setup (test_acceptance.py:264-297, fewer epochs):
  the pre-trained parameters and normalizer it starts from, every step's
  source batch and same-leaf-count target draw (recorded by wrapping
  `costmodel.backward`), and the per-epoch log (train loss, CMD, val MAPE).
* domain.npz — the Box-Cox domain edge (dataset.py:103-105): a normalizer
  whose decode leaves the domain for the untrained desk model's
  predictions; the reference's `predict_batch` raises DomainError and its
  `train` logs val MAPE = inf (`_evaluate`, costmodel.py:658-665).

Like make_golden.py this runs in the build container only; the fixtures
are committed and nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from tpcost import costmodel as cm  # noqa: E402
from tpcost.dataset import (DEFAULT_SYNTH_DEVICE, BoxCoxNormalizer,  # noqa: E402
                            SynthOracleConfig, generate_synthetic, split_dataset)
from tpcost.errors import DomainError  # noqa: E402
from tpcost.features import CompactAst, encode_input  # noqa: E402

DEVICES = {DEFAULT_SYNTH_DEVICE.name: DEFAULT_SYNTH_DEVICE}
SPLIT = {"train": 0, "valid": 1, "test": 2}


def shift_compact(compact, delta=2.0, lo=10, hi=15):
    """test_acceptance.py:264-268"""
    vecs = compact.leaf_vectors.copy()
    vecs[:, lo:hi + 1] += delta
    return CompactAst(leaf_vectors=vecs, ordering=compact.ordering,
                      serialized=compact.serialized, n_leaf=compact.n_leaf)


def compacts(samples):
    return dict(vectors=np.concatenate([s.compact.leaf_vectors for s in samples]),
                ordering=np.concatenate([np.array(s.compact.ordering) for s in samples]),
                n_leaf=np.array([s.compact.n_leaf for s in samples]),
                latency=np.array([s.latency_s for s in samples]))


def norm_blob(nrm):
    return np.array([nrm.lambda_bc, nrm.shift, nrm.t_mean, nrm.t_std, nrm.loss_offset])


def finetune_fixture():
    ds = split_dataset(generate_synthetic(800, [DEFAULT_SYNTH_DEVICE],
                                          SynthOracleConfig(noise_sigma=0.0), seed=100), seed=0)
    pre = cm.train(cm.desk_config(epochs=4, seed=0), ds, DEVICES)
    tgt_samples = ds.subset("test") + ds.subset("valid")
    target_inputs = [encode_input(shift_compact(s.compact), DEFAULT_SYNTH_DEVICE)
                     for s in tgt_samples]
    config = cm.desk_config(epochs=2, seed=0, lr=3e-4, alpha_cmd=1.0)

    # record each step's batches by object identity
    captured = {}
    real_encode, real_backward = cm.encode_dataset, cm.backward
    steps = []

    def encode_spy(samples, devices):
        out = real_encode(samples, devices)
        if "train" not in captured:
            captured["train"] = {id(e): i for i, e in enumerate(out)}
        return out

    tid = {id(e): i for i, e in enumerate(target_inputs)}

    def backward_spy(params, batch, targets, spec, target_batch=None):
        res = real_backward(params, batch, targets, spec, target_batch=target_batch)
        steps.append(([captured["train"][id(e)] for e in batch],
                      [tid[id(e)] for e in (target_batch or [])], res[0], res[2]["cmd"]))
        return res

    cm.encode_dataset, cm.backward = encode_spy, backward_spy
    try:
        tuned = cm.finetune(pre.params, ds, target_inputs, config, DEVICES, pre.normalizer)
    finally:
        cm.encode_dataset, cm.backward = real_encode, real_backward
    src_flat = np.concatenate([np.array(s[0]) for s in steps])
    tgt_flat = np.concatenate([np.array(s[1]) for s in steps])
    out = dict(compacts(ds.samples))
    out.update(split=np.array([SPLIT[ds.splits[s.id]] for s in ds.samples]),
               tgt_rows=np.concatenate([e.matrix for e in target_inputs]),
               tgt_n_leaf=np.array([e.n_leaf for e in target_inputs]),
               norm=norm_blob(pre.normalizer),
               step_src_len=np.array([len(s[0]) for s in steps]),
               step_tgt_len=np.array([len(s[1]) for s in steps]),
               step_src=src_flat, step_tgt=tgt_flat,
               step_loss=np.array([s[2] for s in steps]),
               step_cmd=np.array([s[3] for s in steps]),
               log=np.array([[r.train_loss, r.cmd, r.val_mape, r.val_rmse] for r in tuned.log]))
    out.update({f"T.{k}": np.array(v, copy=True) for k, v in pre.params.tensors.items()})
    np.savez_compressed(OUT / "finetune.npz", **out)


def domain_fixture():
    ds = split_dataset(generate_synthetic(400, [DEFAULT_SYNTH_DEVICE],
                                          SynthOracleConfig(noise_sigma=0.0), seed=7), seed=0)
    lat = np.array([s.latency_s for s in ds.subset("train")])
    # λ = 0.5 puts every transformed label just above the domain edge
    # t = -1/λ = -2 (t = 2·sqrt(y) - 2 for y ~ 1e-6..1e-2), so predictions a
    # little below the labels decode outside the domain
    lam = 0.5
    t = (np.power(lat, lam) - 1.0) / lam
    nrm = BoxCoxNormalizer(lambda_bc=lam, shift=0.0, fitted=True, t_mean=float(t.mean()),
                           t_std=float(t.std()))
    enc_y = nrm.encode(lat)
    nrm.loss_offset = float(max(0.0, -enc_y.min()) + 1.0)
    params = cm.init_params(cm.desk_config(seed=0))
    inputs = cm.encode_dataset(ds.subset("test"), DEVICES)
    pred, _ = cm.forward(params, inputs)
    raised = False
    try:
        cm.predict_batch(params, inputs, nrm)
    except DomainError:
        raised = True
    res = cm.train(cm.desk_config(epochs=1, seed=0), ds, DEVICES, normalizer=nrm)
    vpred, _ = cm.forward(res.params, cm.encode_dataset(ds.subset("valid"), DEVICES))
    base = lam * (vpred * nrm.t_std + nrm.t_mean) + 1.0  # dataset.py:101-105
    print(f"domain fixture: {int((base <= 0).sum())} of {len(base)} validation decodes "
          f"outside the domain (min base {base.min():.3g})")
    out = dict(compacts(ds.samples))
    out.update(split=np.array([SPLIT[ds.splits[s.id]] for s in ds.samples]),
               norm=norm_blob(nrm), test_pred=pred, raised=np.array(raised), val_base=base,
               log=np.array([[r.train_loss, r.val_mape, r.val_rmse] for r in res.log]))
    assert raised and math.isinf(res.log[0].val_mape)
    np.savez_compressed(OUT / "domain.npz", **out)


if __name__ == "__main__":
    finetune_fixture()
    domain_fixture()
    print("round-2 golden fixtures written to", OUT)
