"""Host-side logic that needs no GPU: the batch planner reproduces the
reference's `_epoch_batches` exactly (same RNG calls), the learning-rate
schedule, the Box-Cox fit, and the vectorised synthetic generator's shape."""

import numpy as np
import pytest

from conftest import load_golden


def test_epoch_batches_identical_to_reference():
    from paper_2311_09690_b200.training import epoch_batches
    g = load_golden("plan")
    rng = np.random.default_rng(0)
    for ep in range(2):
        bl = epoch_batches(rng, g["n_leaf"], 64)
        assert np.array_equal(np.concatenate(bl), g[f"ep{ep}.flat"])
        assert np.array_equal(np.array([len(b) for b in bl]), g[f"ep{ep}.len"])
        for b in bl:  # single-bucket batches (costmodel.py:639-643)
            assert len(set(g["n_leaf"][b].tolist())) == 1


def test_lr_schedule_shapes():
    from paper_2311_09690_b200 import desk_config
    from paper_2311_09690_b200.training import lr_at
    const = desk_config(lr=1e-3, lr_schedule="constant")
    assert lr_at(const, 0) == lr_at(const, 57) == 1e-3
    cyc = desk_config(lr=1e-3, lr_schedule="cyclic")
    assert lr_at(cyc, 0) == pytest.approx(1e-4)
    assert lr_at(cyc, 10) == pytest.approx(1e-3)
    assert lr_at(cyc, 5) == pytest.approx((1e-4 + 1e-3) / 2)


def test_fit_boxcox_matches_reference_normalizer():
    from paper_2311_09690_b200.dataset import fit_boxcox
    g = load_golden("c1_4096")
    gm = load_golden("model_desk")
    y = g["latency"][g["split"] == 0]
    norm = fit_boxcox(y)
    lam, shift, tm, ts, off = gm["norm"]
    assert norm.lambda_bc == pytest.approx(lam, abs=1e-12)
    assert norm.t_mean == pytest.approx(tm, rel=1e-12)
    assert norm.t_std == pytest.approx(ts, rel=1e-12)
    assert norm.loss_offset == pytest.approx(off, rel=1e-12)
    assert np.allclose(norm.decode(norm.encode(y)), y, rtol=1e-10)


def test_init_params_bit_identical_to_reference():
    import hashlib
    from paper_2311_09690_b200 import desk_config, init_params
    gm = load_golden("model_desk")
    h = hashlib.sha256()
    for k, v in init_params(desk_config(seed=0)).tensors.items():
        h.update(k.encode())
        h.update(np.ascontiguousarray(v, dtype=np.float64).tobytes())
    assert h.hexdigest() == str(gm["init_sha"])


def test_synthetic_generator_shape():
    from paper_2311_09690_b200 import synth
    s = synth.generate(32768, seed=1)
    assert s.n == 32768 and s.vectors.shape == (int(s.n_leaf.sum()), 24)
    assert s.n_leaf.min() >= 1 and s.n_leaf.max() <= 6
    assert np.all(s.latency > 0)
    ref = load_golden("c1_4096")
    # same generative model: per-column means within a few percent
    m_new, m_ref = s.vectors.mean(0), ref["vectors"].mean(0)
    assert np.all(np.abs(m_new - m_ref) <= 0.15 * np.abs(m_ref) + 0.3)
    tr, va, te = synth.split(327_680)
    assert (len(tr), len(va), len(te)) == (262_144, 32_768, 32_768)
