"""Point-sharded KMeans host logic (sampling.kmeans_sharded) with real
collectives on CPU (gloo, world 1 and 2) and the test-only numpy shard
backend: the k-means++ seeds, the Lloyd assignment (concatenated over the
ranks) and the sizes equal the single-process oracle's; the centres agree
to the last few ulps (the rank split regroups the member sums).  World 1 is
bit-identical.  Includes an empty-cluster repair case."""

import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _data(case):
    rng = np.random.default_rng(11)
    if case == "blobs":
        c = rng.normal(scale=4.0, size=(6, 5))
        x = np.concatenate([c[i] + rng.normal(size=(40, 5)) for i in range(6)])
        return x[rng.permutation(len(x))], 6, None
    # duplicated points + a far one: forces the empty-cluster repair
    x = np.array([[0.0], [0.0], [0.0], [0.0], [0.0], [0.0], [9.0], [9.0]])
    return x, 3, np.array([[0.0], [0.0], [9.0]])


def _worker(rank, world, port, case, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _np_shard import NumpyShard
        from paper_2311_09690_b200.sampling import kmeans_sharded
        x, kappa, init = _data(case)
        parts = np.array_split(np.arange(len(x)), world)
        xl = x[parts[rank]]
        m = kmeans_sharded(xl, kappa, seed=3, init_centers=init,
                           shard=NumpyShard(xl, kappa))
        q.put((rank, m.centers, m.assignment, m.sizes))
    finally:
        dist.destroy_process_group()


def _run(world, case, port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict((r, (c, a, s)) for r, c, a, s in (q.get(timeout=240) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world,case,port", [(1, "blobs", 29631), (2, "blobs", 29632),
                                             (2, "repair", 29633)])
def test_sharded_kmeans_matches_single_process_oracle(world, case, port):
    sys.path.insert(0, ROOT)
    from oracle import lloyd
    x, kappa, init = _data(case)
    c_ref, a_ref, s_ref, _ = lloyd.kmeans(x, kappa, seed=3, init_centers=init)
    out = _run(world, case, port)
    a = np.concatenate([out[r][1] for r in range(world)])
    assert np.array_equal(a, a_ref)
    for r in range(world):
        assert np.array_equal(out[r][2], s_ref)
        assert np.array_equal(out[r][0], out[0][0])  # replicated centres, bitwise
        if world == 1:
            assert np.array_equal(out[r][0], c_ref)
        else:
            assert np.allclose(out[r][0], c_ref, rtol=1e-13, atol=1e-13)
