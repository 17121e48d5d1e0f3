"""Data-parallel CMD fine-tuning step on CPU with real collectives (gloo,
world 2) — the contract of the device trainer's CMD path (capi_train.cu
run_step): every rank writes its source / target latent rows
at their global positions (src_pos, ns_glob + tgt_pos of the step table) of
a zeroed [zs; zt] matrix, one all-reduce SUM assembles the global matrix in
the reference's input order, every rank evaluates the CMD statistics over
it and back-propagates the rows it owns; the gradient all-reduce then gives
exactly the single-process `backward(..., target_batch)` gradient
(costmodel.py:529-570), including the support gradient routed to the FIRST
argmax / argmin row of the union when the extreme value is tied across
ranks (costmodel.py:476-485)."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALPHA = 1.0


def _problem():
    from oracle import predictor as op
    dm = op.Dims(8, 1, 2, 8, 6, 3, (6,), 4)
    prng = np.random.default_rng(1)
    T = {n: prng.normal(scale=0.3, size=s) for n, s in op.tensor_specs(dm)}
    X = prng.normal(size=(300, 4, 24))
    dev = prng.normal(size=(300, 6))
    Y = prng.uniform(1, 3, size=300)
    Xt = prng.normal(0.3, 1.2, size=(120, 4, 24))
    devt = prng.normal(size=(120, 6))
    rng = np.random.default_rng(5)
    n_leaf = rng.integers(1, 5, size=300)
    tgt_leaf = rng.integers(1, 5, size=120)
    tb = {}
    for i, L in enumerate(tgt_leaf.tolist()):
        tb.setdefault(L, []).append(i)
    tb = {k: np.asarray(v) for k, v in tb.items()}
    return dm, T, X, dev, Y, Xt, devt, n_leaf, tgt_leaf, tb


def _grad_step(T, dm, X, dev, Y, Xt, devt, src, tgt, L, n_norm, cmd_rows):
    """Oracle backward of this rank's share: hybrid-free MSE normalised by
    the global batch plus α·dCMD on the rows it owns.  cmd_rows(zs, zt) →
    (value, gs_own, gt_own) evaluates CMD over the assembled global matrix."""
    from oracle import predictor as op
    names = [n for n, _ in op.tensor_specs(dm)]
    G = {}
    zs = np.zeros((0, dm.d_embed))
    zt = np.zeros((0, dm.d_embed))
    tape_s = tape_t = None
    if len(src):
        pred, _, _, zs, tape_s = op.bucket_forward(T, dm, X[src, :L], dev[src])
    if len(tgt):
        _, _, _, zt, tape_t = op.bucket_forward(T, dm, Xt[tgt, :L], devt[tgt])
    value, gs, gt = cmd_rows(zs, zt)
    if len(src):
        op.bucket_backward(T, dm, tape_s, 2.0 * (pred - Y[src]) / n_norm, ALPHA * gs, G)
    if len(tgt):
        op.bucket_backward(T, dm, tape_t, np.zeros(len(tgt)), ALPHA * gt, G)
    return value, np.concatenate([G.get(n, np.zeros_like(T[n])).ravel() for n in names])


def _tied_matrix():
    """[zs (10 rows); zt (6 rows)] with the column-0 maximum tied between
    row 2 (rank 0's share) and row 7 (rank 1's), the column-1 minimum tied
    between target rows 1 and 4 (ranks 0 and 1)."""
    r = np.random.default_rng(3)
    z = r.normal(size=(16, 5))
    z[2, 0] = z[7, 0] = 9.0
    z[10 + 1, 1] = z[10 + 4, 1] = -9.0
    return z


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import moments as om
        from paper_2311_09690_b200.training import plan_epoch
        dm, T, X, dev, Y, Xt, devt, n_leaf, tgt_leaf, tb = _problem()
        flat, steps = plan_epoch(np.random.default_rng(9), n_leaf, 8, world, rank, tb,
                                 len(tgt_leaf))
        out = []
        for k in range(3):
            o, ns, nt, n_norm, sp, nsg, tp, ntg = (int(v) for v in steps[k])
            src, tgt = flat[o:o + ns], flat[o + ns:o + ns + nt]
            L = int(n_leaf[src[0]]) if ns else int(tgt_leaf[tgt[0]])

            def cmd_rows(zs, zt):
                zall = torch.zeros((nsg + ntg, dm.d_embed), dtype=torch.float64)
                zall[sp:sp + ns] = torch.from_numpy(zs)
                zall[nsg + tp:nsg + tp + nt] = torch.from_numpy(zt)
                dist.all_reduce(zall)  # assembles the global [zs; zt]
                z = zall.numpy()
                v, gs, gt = om.cmd_grad(z[:nsg], z[nsg:], 5)
                return v, gs[sp:sp + ns], gt[tp:tp + nt]

            value, g = _grad_step(T, dm, X, dev, Y, Xt, devt, src, tgt, L, n_norm, cmd_rows)
            t = torch.from_numpy(g)
            dist.all_reduce(t)
            out.append((value, t.numpy()))
        # tie routing across ranks on a crafted matrix
        z = _tied_matrix()
        own_s = slice(0, 5) if rank == 0 else slice(5, 10)
        own_t = slice(0, 3) if rank == 0 else slice(3, 6)
        zall = torch.zeros_like(torch.from_numpy(z))
        zall[own_s] = torch.from_numpy(z[own_s])
        zall[10 + own_t.start:10 + own_t.stop] = torch.from_numpy(z[10 + own_t.start:10 + own_t.stop])
        dist.all_reduce(zall)
        v, gs, gt = om.cmd_grad(zall.numpy()[:10], zall.numpy()[10:], 5)
        q.put((rank, out, (v, gs[own_s], gt[own_t])))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(240)
def test_dp_cmd_step_equals_single_process():
    world = 2
    port = 31500 + (os.getpid() % 2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=200) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    from oracle import moments as om
    from paper_2311_09690_b200.training import plan_epoch
    dm, T, X, dev, Y, Xt, devt, n_leaf, tgt_leaf, tb = _problem()
    flat, steps = plan_epoch(np.random.default_rng(9), n_leaf, 8 * world, 1, 0, tb,
                             len(tgt_leaf))
    for k in range(3):
        o, ns, nt, n_norm = (int(v) for v in steps[k][:4])
        src, tgt = flat[o:o + ns], flat[o + ns:o + ns + nt]
        L = int(n_leaf[src[0]])
        assert nt > 0 and ns > 1

        def cmd_rows(zs, zt):
            return om.cmd_grad(zs, zt, 5)

        want_v, want_g = _grad_step(T, dm, X, dev, Y, Xt, devt, src, tgt, L, n_norm, cmd_rows)
        for r in res:  # every rank sees the global CMD value and the global gradient
            assert r[1][k][0] == pytest.approx(want_v, rel=1e-13)
            np.testing.assert_allclose(r[1][k][1], want_g, rtol=1e-11, atol=1e-14)
    # first-index routing of the support gradient when extremes tie across ranks
    z = _tied_matrix()
    v, gs, gt = om.cmd_grad(z[:10], z[10:], 5)
    assert np.count_nonzero(gs[:, 0] - gs[:, 0].mean()) > 0
    got_s = np.vstack([res[0][2][1], res[1][2][1]])
    got_t = np.vstack([res[0][2][2], res[1][2][2]])
    np.testing.assert_array_equal(got_s, gs)
    np.testing.assert_array_equal(got_t, gt)
    assert res[0][2][0] == v == res[1][2][0]
    # the tie is routed to the first row: rows 2 and 7 hold the same column-0
    # value in the same set, so their gradients differ exactly by the support
    # share, which only row 2 (rank 0's) carries; likewise target rows 1 / 4
    assert gs[2, 0] != gs[7, 0] and gt[1, 1] != gt[4, 1]
    others = [r for r in range(10) if r not in (2, 7)]
    assert np.all(gs[others, 0] != gs[2, 0])
