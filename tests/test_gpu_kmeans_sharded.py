"""GPU: point-sharded KMeans (sampling.kmeans_sharded) through the CUDA
shard pieces (tpcb_kmeanspp_closest/_cdf/_search, tpcb_kmeans_partial) and
NCCL collectives.  One GPU here, so world size 1 over NCCL: bit-identical
to the single-device kmeans() (which is bit-exact to the reference).  The
multi-rank orchestration is covered on CPU by test_dist_kmeans.py."""

import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("kappa,seed", [(4, 0), (9, 3)])
def test_sharded_world1_equals_single(pg, kappa, seed):
    from paper_2311_09690_b200 import sampling as s
    g = load_golden("kmeans")
    x = g["cli_x"]
    m1 = s.kmeans(x, kappa, seed=seed)
    m2 = s.kmeans_sharded(x, kappa, seed=seed)
    assert np.array_equal(m1.centers, m2.centers)
    assert np.array_equal(m1.assignment, m2.assignment)
    assert np.array_equal(m1.sizes, m2.sizes)
    assert np.array_equal(m2.centers, g[f"k{kappa}.centers"])


def test_sharded_world1_blobs_and_repair(pg):
    from paper_2311_09690_b200 import sampling as s
    rng = np.random.default_rng(4)
    c = rng.normal(scale=3.0, size=(32, 24))
    x = np.concatenate([c[i] + rng.normal(size=(500, 24)) for i in range(32)])
    x = x[rng.permutation(len(x))]
    for assign in ("exact", "tc"):
        m1 = s.kmeans(x, 32, seed=1, assign=assign)
        m2 = s.kmeans_sharded(x, 32, seed=1, assign=assign)
        assert np.array_equal(m1.centers, m2.centers)
        assert np.array_equal(m1.assignment, m2.assignment)
    x = np.array([[0.0], [0.0], [0.0], [0.0], [9.0], [9.0]])
    init = np.array([[0.0], [0.0], [9.0]])
    m1 = s.kmeans(x, 3, init_centers=init)
    m2 = s.kmeans_sharded(x, 3, init_centers=init)
    assert np.array_equal(m1.assignment, m2.assignment) and min(m2.sizes) >= 1
