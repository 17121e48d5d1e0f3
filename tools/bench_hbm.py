"""HBM-bound kernels at full scale ("report their HBM fraction at
full scale"): K1 featurize+pack, grid CMD (cmd_between), Adam at the
full_reference_config parameter count.

    python tools/bench_hbm.py [--only k1|cmd|adam]

Each: CUDA events on the launching stream, L2 flushed (256 MiB write)
before every repetition, median of --reps.  Algorithmic bytes:
  K1   read T·(96 + 4) + 8·(B+1), write T·(96 + 4) + 8·B  (leaf rows without the
       8-float pad, ordering, offsets; row_ast per row, perm + ast_row per AST)
  CMD  3 streaming reads of Z + 1 write of dZ, (ns+nt)·de·8 each (f64)
  Adam 7·4·P (read g, p, m, v; write p, m, v)
One JSON line per kernel; `peak` is MEASURED_PEAKS.json hbm_gbs.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]


def timed(fn, reps, flush):
    s = torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


def line(metric, ms, alg, **kw):
    gbs = alg / ms / 1e6
    d = {"metric": metric, "ms": ms, "alg_bytes": alg, "achieved_gbs": gbs, "peak_gbs": PEAK,
         "frac": gbs / PEAK, "l2": "flushed"}
    d.update(kw)
    print(json.dumps(d), flush=True)


def bench_k1(reps, flush):
    from paper_2311_09690_b200 import engine, synth
    data = synth.generate(1 << 20, seed=0)
    rows = torch.from_numpy(data.vectors.astype(np.float32)).cuda()
    order = torch.from_numpy(data.ordering).cuda()
    off = torch.from_numpy(data.offsets()).cuda()
    st = engine.Status(rows.device)
    B, T = data.n, int(data.n_leaf.sum())
    pk = engine.pack(rows, order, off, B, 16, False, st, 64)
    ms = timed(lambda: engine.pack(rows, order, off, B, 16, False, st, 64, out=pk), reps, flush)
    st.check("pack")
    alg = T * (96 + 4) + 8 * (B + 1) + T * (96 + 4) + 8 * B
    line("K1 featurize+pack (1,048,576 synthetic ASTs, f32 rows, R=64)", ms, alg, n_ast=B,
         n_tok=T, asts_per_s=B / ms * 1e3)


def bench_cmd(reps, flush):
    from paper_2311_09690_b200 import _lib, engine
    lib = _lib.load()
    ns, nt, de, k = 262144, 65536, 32, 5
    rng = np.random.default_rng(0)
    z = torch.from_numpy(np.vstack([rng.normal(size=(ns, de)),
                                    rng.normal(0.3, 1.2, size=(nt, de))])).cuda()
    val = torch.zeros(1, dtype=torch.float64, device="cuda")
    grad = torch.empty_like(z)
    ws = torch.empty(int(lib.tpcb_cmd_grid_ws(ns, nt, de, k)), dtype=torch.uint8, device="cuda")

    def run_grid():
        _lib.check(lib.tpcb_cmd_grid(z.data_ptr(), 1, ns, nt, de, k, val.data_ptr(),
                                     grad.data_ptr(), ws.data_ptr(), ws.numel(),
                                     engine.stream_ptr()), "cmd_grid")

    def run_one():
        _lib.check(lib.tpcb_cmd(z.data_ptr(), 1, ns, nt, de, k, val.data_ptr(), grad.data_ptr(),
                                engine.stream_ptr()), "cmd")
    run_grid()
    ms = timed(run_grid, reps, flush)
    v_grid = float(val.item())
    ms1 = timed(run_one, max(2, reps // 5), flush)
    v_one = float(val.item())
    n = (ns + nt) * de * 8
    line("CMD grid (cmd_between: 262,144 + 65,536 rows x 32, f64, value + gradient)", ms, 4 * n,
         single_cta_ms=ms1, value_grid=v_grid, value_single_cta=v_one)


def bench_adam(reps, flush):
    from paper_2311_09690_b200 import _lib, engine
    lib = _lib.load()
    P = 46_694_875  # full_reference_config parameter count
    g = torch.randn(P, device="cuda") * 1e-3
    p = torch.randn(P, device="cuda")
    m = torch.zeros(P, device="cuda")
    v = torch.zeros(P, device="cuda")
    opt = _lib.OptimCfg(1, 0.9, 0.999, 1e-8, 0.0)

    def run():
        _lib.check(lib.tpcb_optimizer_step(None, P, p.data_ptr(), None, g.data_ptr(),
                                           m.data_ptr(), v.data_ptr(), C.byref(opt), 1e-3, 1,
                                           engine.stream_ptr()), "adam")
    run()
    ms = timed(run, reps, flush)
    line("Adam step (P = 46,694,875, full_reference_config; fp32 p/m/v)", ms, 7 * 4 * P, params=P)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, fn in (("k1", bench_k1), ("cmd", bench_cmd), ("adam", bench_adam)):
        if not a.only or a.only == name:
            fn(a.reps, flush)


if __name__ == "__main__":
    main()
