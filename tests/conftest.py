import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class _Eager(dict):
    """npz contents loaded once (NpzFile re-inflates a member per access)."""

    @property
    def files(self):
        return list(self.keys())


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return _Eager({k: z[k] for k in z.files})


class GoldenModel:
    """Config + tensors + inputs of a tests/golden/model_*.npz fixture."""

    def __init__(self, name):
        z = load_golden(f"model_{name}")
        self.z = z
        self.cfg = dict(d_model=int(z["d_model"]), n_layers=int(z["n_layers"]),
                        n_heads=int(z["n_heads"]), d_ff=int(z["d_ff"]),
                        d_embed=int(z["d_embed"]), d_device=int(z["d_device"]),
                        decoder_dims=tuple(int(v) for v in z["decoder_dims"]),
                        n_leaf_max=int(z["n_leaf_max"]), seed=int(z["seed"]))
        self.T = {k[2:]: z[k] for k in z.files if k.startswith("T.")}

    def rows(self, prefix):
        z = self.z
        n_leaf = z[f"{prefix}_n_leaf"]
        rows = z[f"{prefix}_rows"]
        off = np.concatenate([[0], np.cumsum(n_leaf)])
        return [rows[off[i]:off[i + 1]] for i in range(len(n_leaf))], z[f"{prefix}_dev"]

    def grads(self, case):
        pre = f"bw.{case}.G."
        return {k[len(pre):]: self.z[k] for k in self.z.files if k.startswith(pre)}


@pytest.fixture(scope="session")
def golden_model():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = GoldenModel(name)
        return cache[name]
    return get


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
