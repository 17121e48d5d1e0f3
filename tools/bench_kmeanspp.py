"""k-means++ seeding (K10, sampling._kmeans_pp_init) at C4 scale.

    python tools/bench_kmeanspp.py [--n 1048576] [--d 32] [--k 1024]

Times DeviceKMeans.kmeanspp (wall clock, synchronised) on Gaussian-blob data
and prints one JSON line with the per-step time and the algorithmic bytes per
step (x read once + closest read/write + the CDF pass: n·d·8 + 4·n·8).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--d", type=int, default=32)
    ap.add_argument("--k", type=int, default=1024)
    a = ap.parse_args()
    from paper_2311_09690_b200.sampling import DeviceKMeans
    rng = np.random.default_rng(0)
    centers = rng.normal(0, 4, size=(64, a.d))
    x = centers[rng.integers(0, 64, a.n)] + rng.normal(size=(a.n, a.d))
    km = DeviceKMeans(np.ascontiguousarray(x), a.k)
    km.kmeanspp(np.random.default_rng(1))  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    km.kmeanspp(np.random.default_rng(1))
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    per = t / (a.k - 1)
    alg = a.n * a.d * 8 + 4 * a.n * 8
    print(json.dumps({"metric": f"k-means++ {a.n}x{a.k} d{a.d}", "s": t, "us_per_step": per * 1e6,
                      "alg_bytes_per_step": alg, "achieved_gbs": alg / per / 1e9}))


if __name__ == "__main__":
    main()
