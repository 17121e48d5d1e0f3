"""K0 (device compact-AST builder) throughput and the trees → latency chain.

    python tools/bench_compact.py [--n 1048576]

Builds a synthetic-shaped forest directly as arrays (a root loop over 1..6
per-leaf chains of 1..3 loops, extents 1..512, the generate_synthetic shape,
dataset.py:312-382), then times with CUDA events on the launching stream:
  * tpcb_build_compact alone (inputs resident in HBM), algorithmic bytes
    = node arrays read (8+4+1 B/node + 8 B offsets) + stats read (72 B/leaf)
    + vectors/ordering written (196 B/leaf) + serialized written (4 B/entry);
  * predict_forest: H2D of the forest + K0 + K1 + fused forward (+ decode).
Prints one JSON line per measurement.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def synth_forest(n: int, seed: int = 0):
    from paper_2311_09690_b200.forest import FlatForest
    rng = np.random.default_rng(seed)
    L = rng.integers(1, 7, n)
    leaf_prog = np.repeat(np.arange(n), L)
    c = rng.integers(1, 4, leaf_prog.size)             # chain loops per leaf
    seg = c + 1                                        # nodes per leaf segment
    nodes_per_prog = 1 + np.bincount(leaf_prog, weights=seg, minlength=n).astype(np.int64)
    node_off = np.concatenate([[0], np.cumsum(nodes_per_prog)])
    leaf_off = np.concatenate([[0], np.cumsum(L)])
    first_leaf = leaf_off[:-1][leaf_prog]
    seg_cum = np.cumsum(seg) - seg                     # global exclusive cumsum
    seg_start = 1 + seg_cum - (np.cumsum(seg) - seg)[first_leaf]  # local start in program
    N = int(node_off[-1])
    parent = np.empty(N, dtype=np.int32)
    extent = np.empty(N, dtype=np.int64)
    annot = np.zeros(N, dtype=np.uint8)
    roots = node_off[:-1]
    parent[roots] = -1
    extent[roots] = rng.integers(4, 64, n)
    seg_node0 = roots[leaf_prog] + seg_start
    j = np.arange(int(seg.sum())) - np.repeat(np.cumsum(seg) - seg, seg)
    gidx = np.repeat(seg_node0, seg) + j
    local0 = np.repeat(seg_start, seg)
    parent[gidx] = np.where(j == 0, 0, local0 + j - 1)
    is_leaf = j == np.repeat(c, seg)
    extent[gidx] = np.where(is_leaf, 0, rng.integers(1, 513, gidx.size))
    annot[gidx] = np.where(is_leaf, 0, rng.integers(0, 8, gidx.size))
    stats = np.stack([rng.integers(1, 513, L.sum()), rng.integers(0, 33, L.sum()),
                      rng.integers(0, 33, L.sum()), rng.integers(0, 3, L.sum()),
                      rng.integers(0, 3, L.sum()), 4 * rng.integers(1, 33, L.sum()),
                      4 * rng.integers(1, 9, L.sum()), rng.integers(1, 5, L.sum()),
                      rng.integers(1, 3, L.sum())], axis=1).astype(np.int64)
    return FlatForest(node_off=node_off.astype(np.int64), parent=parent, extent=extent,
                      annot=annot, leaf_off=leaf_off.astype(np.int64), stats=stats)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import _lib, engine
    from paper_2311_09690_b200.forest import build_compact, predict_forest
    f = synth_forest(a.n)
    f.validate()
    lib = _lib.load()
    dc = build_compact(f)  # warm + allocate
    up = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    args = [up(f.node_off), up(f.parent), up(f.extent), up(f.annot), up(f.leaf_off), up(f.stats)]
    bad = torch.empty(1, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    times = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        lib.tpcb_build_compact(*[t.data_ptr() for t in args], f.n_prog, dc.vectors.data_ptr(),
                               dc.ordering.data_ptr(), dc.serialized.data_ptr(), bad.data_ptr(),
                               engine.stream_ptr())
        e1.record(s)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    N, NL = f.n_nodes, f.n_leaves
    alg = N * 13 + 2 * (f.n_prog + 1) * 8 + NL * 72 + NL * (192 + 4) + (N + NL) * 4
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
    print(json.dumps({"metric": "K0 build_compact programs/s", "n_prog": f.n_prog, "nodes": N,
                      "leaves": NL, "ms": ms, "value": f.n_prog / ms * 1e3,
                      "alg_bytes": alg, "gbs": alg / ms / 1e6,
                      "hbm_frac": alg / ms / 1e6 / peaks["hbm_gbs"], "l2": "flushed"}))
    params = pb.init_params(pb.desk_config(seed=0))
    pred = pb.Predictor(params)
    dev = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    predict_forest(pred, f, dev, None, validate=False)
    torch.cuda.synchronize()
    import time
    t = []
    for _ in range(5):
        t0 = time.perf_counter()
        predict_forest(pred, f, dev, None, validate=False)
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    ts = float(np.median(t))
    print(json.dumps({"metric": "predict_forest trees->latency programs/s (host arrays in, "
                      "host latencies out)", "n_prog": f.n_prog, "s": ts,
                      "value": f.n_prog / ts}))


if __name__ == "__main__":
    main()
