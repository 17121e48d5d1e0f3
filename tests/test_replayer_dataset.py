"""Dataset persistence (reference JSONL, dataset.py:421-485, and the binary
ragged SoA) and the batched replayer.dedup_predict (replayer.py:175-198)."""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

REF_JSONL = GOLDEN / "dataset_ref.jsonl"


def test_jsonl_reader_writer_byte_identical_to_reference(tmp_path):
    import paper_2311_09690_b200 as pb
    ds = pb.load_dataset(REF_JSONL)
    assert len(ds.samples) == 40
    out = tmp_path / "again.jsonl"
    pb.save_dataset(ds, out)
    assert out.read_bytes() == REF_JSONL.read_bytes()


def test_binary_dataset_roundtrip_exact(tmp_path):
    import paper_2311_09690_b200 as pb
    ds = pb.split_dataset(pb.load_dataset(REF_JSONL), seed=1)
    path = tmp_path / "ds.npz"
    pb.save_dataset_bin(ds, path)
    back = pb.load_dataset_bin(path)
    assert back.splits == ds.splits
    for a, b in zip(ds.samples, back.samples):
        assert (a.id, a.task_id, a.model_id, a.device_id) == (b.id, b.task_id, b.model_id,
                                                              b.device_id)
        assert a.compact == b.compact and a.latency_s == b.latency_s
    # JSONL of the binary copy is byte-identical too
    pb.save_dataset(back, tmp_path / "b.jsonl")
    assert (tmp_path / "b.jsonl").read_bytes() == REF_JSONL.read_bytes()


def test_binary_dataset_loads_as_compact_batch(tmp_path):
    import paper_2311_09690_b200 as pb
    ds = pb.load_dataset(REF_JSONL)
    path = tmp_path / "ds.npz"
    pb.save_dataset_bin(ds, path)
    dev = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    batch, y, split, ids = pb.load_batch_bin(path, {"synth0": dev})
    want = pb.CompactBatch.from_compacts([s.compact for s in ds.samples], dev, dtype=np.float64)
    assert np.array_equal(batch.vectors, want.vectors)
    assert np.array_equal(batch.ordering, want.ordering)
    assert np.array_equal(batch.n_leaf, want.n_leaf)
    assert np.array_equal(batch.device_features(), want.device_features())
    assert np.array_equal(y, ds.labels())
    with pytest.raises(pb.errors.ValidationError):
        pb.load_batch_bin(path, {"other": dev})


def test_dedup_predict_custom_predictor_semantics():
    """Reference semantics (replayer.py:175-198) with a custom predictor: one
    call per distinct key in first-seen order, every node filled, missing
    program → ValidationError."""
    import paper_2311_09690_b200 as pb
    calls = []

    def fake(compact, dev):
        calls.append(compact)
        return 10.0 * compact
    nodes = [SimpleNamespace(tir_key=k, duration=None) for k in "abcab"]
    d = pb.dedup_predict(SimpleNamespace(nodes=nodes), {"a": 1, "b": 2, "c": 3}, None, "dev",
                         None, predictor=fake)
    assert d == {"a": 10.0, "b": 20.0, "c": 30.0} and calls == [1, 2, 3]
    assert [n.duration for n in nodes] == [10.0, 20.0, 30.0, 10.0, 20.0]
    with pytest.raises(pb.errors.ValidationError):
        pb.dedup_predict(SimpleNamespace(nodes=nodes), {"a": 1}, None, "dev", None,
                         predictor=fake)


@pytest.mark.gpu
def test_dedup_predict_batched_matches_per_key_and_reference(golden_model):
    """One device batch over the distinct keys equals the per-key predict
    calls bit for bit, and the reference's decoded latencies within 1e-3."""
    import paper_2311_09690_b200 as pb
    gm = golden_model("desk")
    c = gm.cfg
    cfg = pb.CostModelConfig(**c)
    params = pb.CostModelParams(cfg, gm.T)
    lam, shift, tm, ts, off = gm.z["norm"]
    norm = pb.BoxCoxNormalizer(lam, shift, True, tm, ts, off)
    c1 = load_golden("c1_4096")
    noff = np.concatenate([[0], np.cumsum(c1["n_leaf"])])
    synth = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    idx = list(range(0, 4096, 97))
    programs = {f"k{i}": pb.CompactAst(c1["vectors"][noff[i]:noff[i + 1]],
                                       tuple(c1["ordering"][noff[i]:noff[i + 1]].tolist()), (),
                                       int(c1["n_leaf"][i])) for i in idx}
    order = [f"k{i}" for i in idx] * 3
    np.random.default_rng(0).shuffle(order)
    nodes = [SimpleNamespace(tir_key=k, duration=None) for k in order]
    d = pb.dedup_predict(SimpleNamespace(nodes=nodes), programs, params, synth, norm)
    assert len(d) == len(idx)
    per_key = {k: pb.predict(params, programs[k], synth, norm) for k in list(programs)[:6]}
    for k, v in per_key.items():
        assert d[k] == v
    want = {f"k{i}": gm.z["latency4k"][i] for i in idx}
    rel = max(abs(d[k] - want[k]) / want[k] for k in d)
    assert rel <= 1e-3, rel
    assert all(n.duration == d[n.tir_key] for n in nodes)
