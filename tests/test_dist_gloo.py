"""Data-parallel host logic on CPU with real collectives (gloo, world 2):
the per-rank epoch plans partition the global plan exactly, and the
per-rank gradients (oracle arithmetic, loss normalised by the global batch)
all-reduce to the single-process full-batch gradient — the contract the
device trainer's NCCL all-reduce relies on (training.py / capi_train.cu)."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q, mode):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import predictor as op
        from paper_2311_09690_b200.training import plan_epoch
        rng = np.random.default_rng(5)
        n_leaf = rng.integers(1, 5, size=300)
        tgt_leaf = rng.integers(1, 5, size=120)
        tb = {}
        for i, L in enumerate(tgt_leaf.tolist()):
            tb.setdefault(L, []).append(i)
        tb = {k: np.asarray(v) for k, v in tb.items()}
        # weak: 8 per rank (global 16); strong: the global batch of 16 split
        flat, steps = plan_epoch(np.random.default_rng(9), n_leaf, 8 if mode == "weak" else 16,
                                 world, rank, tb, len(tgt_leaf), dp_mode=mode)
        # gather every rank's plan
        gathered = [None] * world
        dist.all_gather_object(gathered, (flat.tolist(), steps.tolist()))
        # gradient check on one step with the oracle (tiny config)
        dm = op.Dims(8, 1, 2, 8, 6, 3, (6,), 4)
        prng = np.random.default_rng(1)
        T = {n: prng.normal(scale=0.3, size=s) for n, s in op.tensor_specs(dm)}
        X = prng.normal(size=(300, 4, 24))
        dev = prng.normal(size=(300, 6))
        Y = prng.uniform(1, 3, size=300)
        o, ns, _, n_norm = steps[0][:4]
        mine = flat[o:o + ns]
        L = int(n_leaf[mine[0]]) if ns else 1
        G = {}
        if ns:
            pred, _, _, _, tape = op.bucket_forward(T, dm, X[mine, :L], dev[mine])
            d = pred - Y[mine]
            dpred = 2.0 * d / n_norm  # global normalisation
            op.bucket_backward(T, dm, tape, dpred, None, G)
        names = [n for n, _ in op.tensor_specs(dm)]
        vec = np.concatenate([G.get(n, np.zeros_like(T[n])).ravel() for n in names])
        t = torch.from_numpy(vec)
        dist.all_reduce(t)
        q.put((rank, gathered, t.numpy(), L))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(240)
@pytest.mark.parametrize("mode", ["weak", "strong"])
def test_dp_plan_partition_and_gradient_allreduce(mode):
    """Both data-parallel modes: "weak" (8 per rank, global batch 16) and
    "strong" (the global batch of 16 split across the ranks) partition the
    same world-1 plan of batch 16 — strong keeps the reference's step count
    for its batch size at any world size."""
    world = 2
    port = 29500 + (os.getpid() % 2000) + (0 if mode == "weak" else 7)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=200) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    from oracle import predictor as op
    from paper_2311_09690_b200.training import plan_epoch
    rank0 = [r for r in res if r[0] == 0][0]
    gathered = rank0[1]
    rng = np.random.default_rng(5)
    n_leaf = rng.integers(1, 5, size=300)
    tgt_leaf = rng.integers(1, 5, size=120)
    tb = {}
    for i, L in enumerate(tgt_leaf.tolist()):
        tb.setdefault(L, []).append(i)
    tb = {k: np.asarray(v) for k, v in tb.items()}
    full_flat, full_steps = plan_epoch(np.random.default_rng(9), n_leaf, 8 * world, 1, 0, tb,
                                       len(tgt_leaf))
    if mode == "strong":  # the reference's own batching at batch size 16
        from paper_2311_09690_b200.training import epoch_batches
        assert len(full_steps) == len(epoch_batches(np.random.default_rng(9), n_leaf, 16))
    plans = [(np.array(f, dtype=np.int64), np.array(s)) for f, s in gathered]
    assert all(len(p[1]) == len(full_steps) for p in plans)
    for k, (o, ns, nt, n_norm, sp, nsg, tp, ntg) in enumerate(full_steps):
        want_s = full_flat[o:o + ns]
        want_t = full_flat[o + ns:o + ns + nt]
        got_s = np.concatenate([p[0][p[1][k][0]:p[1][k][0] + p[1][k][1]] for p in plans])
        got_t = np.concatenate([p[0][p[1][k][0] + p[1][k][1]:p[1][k][0] + p[1][k][1] + p[1][k][2]]
                                for p in plans])
        assert np.array_equal(got_s, want_s) and np.array_equal(got_t, want_t)
        for p in plans:  # positions and global counts consistent
            assert p[1][k][3] == ns and p[1][k][5] == ns and p[1][k][7] == nt
        assert plans[1][1][k][4] == plans[0][1][k][1]
    # all-reduced per-rank gradients == single-process full-batch gradient
    dm = op.Dims(8, 1, 2, 8, 6, 3, (6,), 4)
    prng = np.random.default_rng(1)
    T = {n: prng.normal(scale=0.3, size=s) for n, s in op.tensor_specs(dm)}
    X = prng.normal(size=(300, 4, 24))
    dev = prng.normal(size=(300, 6))
    Y = prng.uniform(1, 3, size=300)
    o, ns = full_steps[0][:2]
    b = full_flat[o:o + ns]
    L = rank0[3]
    pred, _, _, _, tape = op.bucket_forward(T, dm, X[b, :L], dev[b])
    G = {}
    op.bucket_backward(T, dm, tape, 2.0 * (pred - Y[b]) / ns, None, G)
    names = [n for n, _ in op.tensor_specs(dm)]
    want = np.concatenate([G.get(n, np.zeros_like(T[n])).ravel() for n in names])
    np.testing.assert_allclose(rank0[2], want, rtol=1e-12, atol=1e-14)
