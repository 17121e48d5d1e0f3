"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (needs /root/reference, read-only):

    python tests/golden/make_golden.py

Nothing on the GPU box reads /root/reference: the fixtures written here are
committed and travel with the repo.  Every fixture is produced by the
reference package `tpcost` itself (pkg/src/tpcost), through its public API
or the private helpers the hot path runs (`_forward`, `_cmd_forward_backward`,
`_kmeans_pp_init`), so the oracle and the CUDA path are pinned to the
reference's own numbers.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from tpcost import costmodel as cm  # noqa: E402
from tpcost import nn as rnn  # noqa: E402
from tpcost import sampling as rs  # noqa: E402
from tpcost.dataset import (DEFAULT_SYNTH_DEVICE, SynthOracleConfig,  # noqa: E402
                            generate_synthetic, split_dataset)
from tpcost.features import (N_ENTRY, CompactAst, DeviceSpec, EncodedInput,  # noqa: E402
                             device_vector, encode_input, positional_encoding)

DEVICES = {DEFAULT_SYNTH_DEVICE.name: DEFAULT_SYNTH_DEVICE}
T4 = DeviceSpec(name="t4", clock_mhz=1590, mem_gb=16, bandwidth_gbps=320,
                cores=40, peak_fp32_gflops=8100, l2_cache_mb=4)

TINY = cm.CostModelConfig(d_model=8, n_layers=1, n_heads=2, d_ff=8,
                          d_embed=6, d_device=3, decoder_dims=(6,),
                          n_leaf_max=3, batch_size=4, epochs=1, seed=0)
GRAD = cm.CostModelConfig(d_model=8, n_layers=1, n_heads=2, d_ff=8,
                          d_embed=6, d_device=3, decoder_dims=(6,),
                          n_leaf_max=2, batch_size=4, epochs=1, seed=20)
MID = cm.CostModelConfig(d_model=16, n_layers=2, n_heads=4, d_ff=24,
                         d_embed=8, d_device=4, decoder_dims=(12, 10),
                         n_leaf_max=7, seed=5)


def cfg_dict(c):
    return dict(d_model=c.d_model, n_layers=c.n_layers, n_heads=c.n_heads,
                d_ff=c.d_ff, d_embed=c.d_embed, d_device=c.d_device,
                decoder_dims=np.array(c.decoder_dims), n_leaf_max=c.n_leaf_max,
                seed=c.seed)


def tensors_blob(prefix, tensors):
    # copies: optimizer steps mutate the reference's tensors in place
    return {f"{prefix}{k}": np.array(v, copy=True) for k, v in tensors.items()}


def tensor_sha(tensors):
    h = hashlib.sha256()
    for k, v in tensors.items():  # creation order
        h.update(k.encode())
        h.update(np.ascontiguousarray(v, dtype=np.float64).tobytes())
    return h.hexdigest()


def ragged(inputs):
    mats = [e.matrix for e in inputs]
    return dict(rows=np.concatenate(mats, axis=0),
                n_leaf=np.array([m.shape[0] for m in mats]),
                dev=np.stack([e.device_vector for e in inputs]))


def compacts_blob(samples):
    return dict(vectors=np.concatenate([s.compact.leaf_vectors for s in samples]),
                ordering=np.concatenate([np.array(s.compact.ordering) for s in samples]),
                n_leaf=np.array([s.compact.n_leaf for s in samples]),
                latency=np.array([s.latency_s for s in samples]),
                task=np.array([int(s.task_id[1:]) for s in samples]),
                model=np.array([int(s.model_id[1:]) for s in samples]))


def group_perm(inputs, n_leaf_max):
    groups = cm._group_by_leaf(inputs, n_leaf_max)
    return np.concatenate([np.array(groups[k]) for k in sorted(groups)])


def rand_inputs(rng, n, leaf_range):
    out = []
    for _ in range(n):
        L = int(rng.integers(*leaf_range))
        out.append(EncodedInput(matrix=rng.normal(size=(L, N_ENTRY)),
                                device_vector=rng.normal(size=6)))
    return out


def backward_cases(params, batch, targets, target_batch, norm_tuple, tag,
                   offset=0.75, keys=None):
    """Reference backward for every LossSpec variant the path supports."""
    out = {}
    specs = {
        "mse": cm.LossSpec(mode="mse"),
        "hyb": cm.LossSpec(mode="hybrid", lambda_hybrid=1e-3, offset=offset),
        "mape": cm.LossSpec(mode="mape", offset=offset),
        "cmd": cm.LossSpec(mode="hybrid", lambda_hybrid=1e-3, offset=offset,
                           alpha_cmd=1.0, cmd_order=5),
        "cmd3": cm.LossSpec(mode="hybrid", lambda_hybrid=1e-3, offset=offset,
                            alpha_cmd=0.5, cmd_order=3),
    }
    if norm_tuple is not None:
        norm = cm.BoxCoxNormalizer(*norm_tuple)
        specs["orig"] = cm.LossSpec(mode="hybrid", lambda_hybrid=0.1,
                                    mape_space="original", normalizer=norm)
    for key, spec in specs.items():
        if keys is not None and key not in keys:
            continue
        tb = target_batch if key.startswith("cmd") else None
        val, grads, aux = cm.backward(params, batch, targets, spec, target_batch=tb)
        out[f"{tag}{key}.loss"] = np.array(val)
        out[f"{tag}{key}.cmd"] = np.array(aux["cmd"])
        for k, v in grads.items():
            if np.any(v != 0.0):  # absent key == all-zero gradient
                out[f"{tag}{key}.G.{k}"] = v
    return out


def main():
    rng = np.random.default_rng(12345)
    # ------------------------------------------------------------ features
    positions = np.array([0, 1, 7, 42, 311, 27, 9000, 3])
    comp = CompactAst(leaf_vectors=np.zeros((len(positions), N_ENTRY)),
                      ordering=tuple(int(p) for p in positions),
                      serialized=tuple(range(9001)), n_leaf=len(positions))
    np.savez_compressed(
        OUT / "features.npz", positions=positions,
        pe=positional_encoding(comp), pe_theta100=positional_encoding(comp, 100.0),
        dev_synth=device_vector(DEFAULT_SYNTH_DEVICE), dev_t4=device_vector(T4))

    # ---------------------------------------------------- synthetic 512 set
    ds = generate_synthetic(512, [DEFAULT_SYNTH_DEVICE],
                            SynthOracleConfig(noise_sigma=0.0), seed=0)
    enc = cm.encode_dataset(ds.samples, DEVICES)
    blob = compacts_blob(ds.samples)
    blob.update({f"enc_{k}": v for k, v in ragged(enc).items()})
    blob["perm"] = group_perm(enc, 16)
    np.savez_compressed(OUT / "synth512.npz", **blob)

    # -------------------------------------- small configs: forward+backward
    for name, cfg, lr_ in (("tiny", TINY, (1, 4)), ("grad", GRAD, (1, 3)),
                           ("mid", MID, (1, 8))):
        params = cm.init_params(cfg)
        local = np.random.default_rng(100 + cfg.seed)
        inputs = rand_inputs(local, 11, lr_)
        tgt_batch = rand_inputs(local, 9, lr_)
        targets = local.uniform(1.0, 3.0, size=len(inputs))
        pred, lat = cm.forward(params, inputs)
        out = cfg_dict(cfg)
        out.update(tensors_blob("T.", params.tensors))
        out.update({f"in_{k}": v for k, v in ragged(inputs).items()})
        out.update({f"tg_{k}": v for k, v in ragged(tgt_batch).items()})
        out.update(targets=targets, pred=pred, z_x=lat.z_x, z_v=lat.z_v, z=lat.z,
                   perm=group_perm(inputs, cfg.n_leaf_max),
                   sha=np.array(tensor_sha(params.tensors)))
        norm_t = (-0.07, 0.0, True, 0.2, 0.9, 1.3)
        out.update(backward_cases(params, inputs, targets, tgt_batch, norm_t, "bw."))
        np.savez_compressed(OUT / f"model_{name}.npz", **out)

    # -------------------------------------------- desk: init + trained ckpt
    desk = cm.desk_config(seed=0)
    init = cm.init_params(desk)
    ds4k = generate_synthetic(4096, [DEFAULT_SYNTH_DEVICE],
                              SynthOracleConfig(noise_sigma=0.0), seed=0)
    sp = split_dataset(ds4k, seed=0)
    res = cm.train(cm.desk_config(epochs=10, seed=0), sp, DEVICES)
    trained = res.params
    nrm = res.normalizer
    enc4k = cm.encode_dataset(ds4k.samples, DEVICES)
    pred_i, lat_i = cm.forward(init, enc)
    pred_t, lat_t = cm.forward(trained, enc4k)
    dec_t = cm.predict_batch(trained, enc4k, nrm)
    out = cfg_dict(desk)
    out.update(tensors_blob("T.", trained.tensors))
    out.update(init_sha=np.array(tensor_sha(init.tensors)),
               init_pred512=pred_i, init_zx512=lat_i.z_x, init_z512=lat_i.z,
               norm=np.array([nrm.lambda_bc, nrm.shift, nrm.t_mean, nrm.t_std,
                              nrm.loss_offset]),
               pred4k=pred_t, z4k=lat_t.z, init_zv512=lat_i.z_v,
               latency4k=dec_t,
               train_log=np.array([[r.train_loss, r.val_mape, r.val_rmse]
                                   for r in res.log]),
               best_epoch=np.array(res.best_epoch))
    # a reference batch (one bucket, 64 samples) + a shifted target batch
    n_leaf = np.array([e.n_leaf for e in enc4k])
    idx = np.flatnonzero(n_leaf == 4)[:64]
    tidx = np.flatnonzero(n_leaf == 4)[64:128]
    batch = [enc4k[i] for i in idx]
    tb = [EncodedInput(matrix=enc4k[i].matrix + np.where(
        (np.arange(N_ENTRY) >= 10) & (np.arange(N_ENTRY) < 16), 2.0, 0.0),
        device_vector=enc4k[i].device_vector) for i in tidx]
    y = nrm.encode(np.array([ds4k.samples[i].latency_s for i in idx]))
    norm_t = (nrm.lambda_bc, nrm.shift, True, nrm.t_mean, nrm.t_std, nrm.loss_offset)
    out.update(batch_idx=idx, tbatch_idx=tidx, batch_y=y)
    out.update(backward_cases(trained, batch, y, tb, norm_t, "bw.",
                              offset=nrm.loss_offset, keys=("hyb", "cmd", "orig")))
    np.savez_compressed(OUT / "model_desk.npz", **out)
    np.savez_compressed(OUT / "c1_4096.npz", **compacts_blob(ds4k.samples),
                        perm=group_perm(enc4k, 16),
                        split=np.array([{"train": 0, "valid": 1, "test": 2}[
                            sp.splits[s.id]] for s in ds4k.samples]))

    # batch planning: the reference's own _epoch_batches on the C1 train split
    tr_nleaf = [s.compact.n_leaf for s in sp.subset("train")]
    prng = np.random.default_rng(0)
    plan = {}
    for ep in range(2):
        bl = cm._epoch_batches(prng, tr_nleaf, 64)
        plan[f"ep{ep}.flat"] = np.concatenate(bl)
        plan[f"ep{ep}.len"] = np.array([len(b) for b in bl])
    np.savez_compressed(OUT / "plan.npz", n_leaf=np.array(tr_nleaf), **plan)

    # acceptance criterion 6 dataset (test_acceptance.py:232-257)
    ds6 = split_dataset(generate_synthetic(2000, [DEFAULT_SYNTH_DEVICE],
                                           SynthOracleConfig(noise_sigma=0.0), seed=11), seed=1)
    np.savez_compressed(OUT / "crit6.npz", **compacts_blob(ds6.samples),
                        split=np.array([{"train": 0, "valid": 1, "test": 2}[ds6.splits[s.id]]
                                        for s in ds6.samples]))

    # ---------------------------------------------------------------- CMD
    out = {}
    crng = np.random.default_rng(2)
    for c in range(12):
        ns, nt = int(crng.integers(2, 40)), int(crng.integers(2, 40))
        d = int(crng.integers(1, 33))
        zs = crng.normal(scale=crng.uniform(0.5, 2.0), size=(ns, d))
        zt = crng.normal(loc=crng.uniform(-1, 1), size=(nt, d))
        if c == 3:  # a column with zero support (floor path)
            zs[:, 0] = 0.25
            zt[:, 0] = 0.25
        if c == 4:  # ties in extrema (first-index routing)
            zs[1] = zs[0]
            zt[0] = zs[0]
        for k in (5, 3):
            v, gs, gt = cm._cmd_forward_backward(zs, zt, k)
            out[f"c{c}.k{k}.value"] = np.array(v)
            out[f"c{c}.k{k}.gs"] = gs
            out[f"c{c}.k{k}.gt"] = gt
        out[f"c{c}.zs"] = zs
        out[f"c{c}.zt"] = zt
    out["hand"] = np.array(cm.cmd(np.array([[0.0], [1.0]]), np.array([[0.5], [0.5]]), 5))
    np.savez_compressed(OUT / "cmd.npz", **out)

    # --------------------------------------------------------------- Adam
    params = cm.init_params(TINY)
    names = list(params.tensors)
    opt = rnn.Adam(names, weight_decay=0.01)
    arng = np.random.default_rng(7)
    out = tensors_blob("p0.", params.tensors)
    for step in range(3):
        grads = {k: arng.normal(size=v.shape) for k, v in params.tensors.items()}
        if step == 1:
            grads[names[3]] = np.zeros_like(grads[names[3]])
        opt.step(params.tensors, grads, 1e-2)
        out.update(tensors_blob(f"g{step}.", grads))
        out.update(tensors_blob(f"p{step + 1}.", params.tensors))
    sgd = rnn.Sgd(names, weight_decay=0.1)
    sgd.step(params.tensors, grads, 0.5)
    out.update(tensors_blob("sgd.", params.tensors))
    np.savez_compressed(OUT / "adam.npz", **out)

    # ------------------------------------------------------------- kmeans
    out = {}
    five = np.array([0.0, 0.1, 5.0, 10.0, 10.1])
    m = rs.kmeans(five, 2, seed=0, init_centers=np.array([0.05, 10.05]))
    out.update(five_centers=m.centers, five_assign=m.assignment, five_sizes=m.sizes)
    xr = np.array([[0.0], [0.0], [0.0], [9.0]])
    m = rs.kmeans(xr, 2, seed=0, init_centers=np.array([[0.0], [0.0]]))
    out.update(rep_centers=m.centers, rep_assign=m.assignment, rep_sizes=m.sizes)
    # blobs: task-structured points like the CLI's mean-pooled leaf vectors
    by_task = {}
    for s in ds.samples:
        by_task.setdefault(s.task_id, []).append(s.compact.leaf_vectors.mean(axis=0))
    task_ids = sorted(by_task)
    tasks = [rs.TaskFeatureSet(t, np.stack(by_task[t])) for t in task_ids]
    x = np.concatenate([t.features for t in tasks], axis=0)
    out["cli_x"] = x
    out["cli_task_rows"] = np.array([len(by_task[t]) for t in task_ids])
    out["cli_task_ids"] = np.array(task_ids)
    for kappa, seed in ((4, 0), (9, 3)):
        krng = np.random.default_rng(seed)
        init_c = rs._kmeans_pp_init(x, kappa, krng)
        mdl = rs.kmeans(x, kappa, seed=seed)
        tbl = rs.build_distance_table(mdl, tasks)
        sel = rs.select_tasks(x, kappa, tasks, seed=seed)
        out.update({f"k{kappa}.init": init_c, f"k{kappa}.centers": mdl.centers,
                    f"k{kappa}.assign": mdl.assignment, f"k{kappa}.sizes": mdl.sizes,
                    f"k{kappa}.psi": tbl.psi, f"k{kappa}.selected": np.array(sel)})
    grng = np.random.default_rng(33)
    blobs = grng.normal(scale=8.0, size=(6, 24))
    xb = np.concatenate([b + grng.normal(scale=1.5, size=(500, 24)) for b in blobs])
    xb = xb[grng.permutation(xb.shape[0])]
    mdl = rs.kmeans(xb, 16, seed=11)
    out.update(blob_x=xb, blob_centers=mdl.centers, blob_assign=mdl.assignment,
               blob_sizes=mdl.sizes,
               blob_init=rs._kmeans_pp_init(xb, 16, np.random.default_rng(11)))
    np.savez_compressed(OUT / "kmeans.npz", **out)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
