"""Secondary measurements of SURVEY §8(d), one JSON line each (B200, 1 GPU):

  C3  CMD fine-tune training throughput: source = the C2 training split,
      target = shifted valid+test (criterion-7 shift), alpha 1, K 5, bs 64+64
  C4  KMeans 1M × 1024 (d = 24 mean-pooled leaf vectors and d = 32 z_x),
      k-means++ + Lloyd to convergence; per-iteration time; exact float64 and
      tensor-core (3xTF32 + exact re-rank) assignment modes
  C5  inference sweep n = 64 … 1M ASTs, fp32 parity mode and bf16 tensor-core mode

  full  full_reference_config (d 716, 11 layers, 46.7 M params) inference
        through the layer-by-layer tensor-core path, and the 3xTF32 GEMM alone
  c4dp  point-sharded KMeans (kmeans_sharded) at the launched world size

python tools/bench_extra.py [c3] [c4] [c4tc] [c5] [c5bf16] [full] [c4dp]  (default: all)
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import engine, synth  # noqa: E402
from paper_2311_09690_b200.dataset import fit_boxcox  # noqa: E402

DSPEC = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
DV = pb.device_vector(DSPEC).astype(np.float32)
SHIFT = np.where((np.arange(24) >= 10) & (np.arange(24) < 16), 2.0, 0.0).astype(np.float32)


def rag(s, shift=None):
    rows = s.vectors.astype(np.float32)
    if shift is not None:
        rows = rows + shift
    return engine.RaggedHost(rows=rows, ordering=s.ordering, n_leaf=s.n_leaf,
                             devfeat=np.tile(DV, (s.n, 1)), encoded=False)


def dev_time(fn, reps=1, stream=None):
    """device time per call, CUDA events on the stream the work runs on"""
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def c3():
    from paper_2311_09690_b200.training import Trainer
    n_gen = 327_680
    data = synth.generate(n_gen, seed=0)
    tr_i, va_i, te_i = synth.split(n_gen, seed=0)
    train = data.take(np.sort(tr_i))
    target = data.take(np.sort(np.concatenate([va_i, te_i])))
    norm = fit_boxcox(train.latency)
    cfg = pb.desk_config(seed=0, alpha_cmd=1.0)
    loss = engine.loss_struct("hybrid", cfg.lambda_hybrid, norm.loss_offset, 1.0, 5,
                              "transformed", norm)
    tr = Trainer(cfg, pb.init_params(cfg).tensors, rag(train), norm.encode(train.latency), loss,
                 target_rag=rag(target, SHIFT))
    rng = np.random.default_rng(0)
    flat, steps = tr.plan(rng)
    tr.run_epoch(cfg.lr, flat, steps)  # warm-up + graph capture
    torch.cuda.synchronize()
    flat, steps = tr.plan(rng)
    t = dev_time(lambda: tr.run_epoch(cfg.lr, flat, steps), stream=tr.stream)
    cmd = tr.step_cmd[:steps.shape[0]].cpu().numpy()
    return {"metric": "C3 CMD fine-tune source samples/s (1 GPU)", "value": train.n / t,
            "unit": "samples/s", "epoch_s": t, "steps": int(steps.shape[0]),
            "batch": "64 source + 64 target (same leaf bucket)", "mean_step_cmd": float(cmd.mean()),
            "dtype": "f32 network, f64 CMD statistics"}


def c4(assign="exact"):
    from paper_2311_09690_b200.sampling import DeviceKMeans
    out = []
    n, k = 1 << 20, 1024
    data = synth.generate(n, seed=0)
    off = data.offsets()
    pooled = np.add.reduceat(data.vectors.astype(np.float64), off[:-1], axis=0) / data.n_leaf[:, None]
    p = pb.Predictor(pb.init_params(pb.desk_config(seed=0)))
    _, zx, _, _, _ = p.forward_ragged(rag(data), None, latents=True)
    for name, x in (("d24 mean-pooled leaf vectors", pooled),
                    ("d32 z_x latents", zx.double().cpu().numpy())):
        km = DeviceKMeans(np.ascontiguousarray(x), k, assign=assign)
        rng = np.random.default_rng(0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        km.kmeanspp(rng)
        torch.cuda.synchronize()
        t_pp = time.perf_counter() - t0
        t_assign = dev_time(km.assign_step, reps=3)
        t0 = time.perf_counter()
        iters = km.lloyd()
        torch.cuda.synchronize()
        t_lloyd = time.perf_counter() - t0
        r = {"metric": f"C4 KMeans {n}x{k} ({name}), {assign} assignment", "kmeanspp_s": t_pp,
             "lloyd_s": t_lloyd, "lloyd_iterations": iters, "assign_pass_ms": t_assign * 1e3}
        if assign == "exact":
            r["assign_fp64_tflops"] = 3.0 * n * k * x.shape[1] / t_assign / 1e12
            r["dtype"] = "f64"
        else:
            r["assign_3xtf32_tflops"] = 3 * 2.0 * n * k * 32 / t_assign / 1e12
            r["dtype"] = "3xTF32 candidates + f64 re-rank"
            ex = DeviceKMeans(np.ascontiguousarray(x), k)
            ex.centers.copy_(km.centers)
            ex.assign_step()
            km.assign_step()
            r["agreement_vs_exact_same_centres"] = float(
                (ex.assign == km.assign).double().mean().item())
        out.append(r)
    return out


def c5(precision="fp32"):
    p = pb.Predictor(pb.init_params(pb.desk_config(seed=0)), precision=precision)
    big = synth.generate(1 << 20, seed=0)
    res = {}
    for n in (64, 256, 1024, 4096, 16384, 65536, 262144, 1 << 20):
        sub = big.take(np.arange(n))
        rows, ordering, leaf_off, devfeat = engine.upload_ragged(rag(sub), torch.device("cuda"))
        f = lambda: p.forward_device(rows, ordering, leaf_off, devfeat, n, False, None,  # noqa
                                     latents=False)
        for _ in range(3):
            f()
        reps = 50 if n <= 65536 else 5
        res[str(n)] = n / dev_time(f, reps)
    mode = {"fp32": "fp32 parity mode (FFMA)",
            "bf16": "bf16 tensor-core mode (tcgen05, fp32 accumulate)"}[precision]
    return {"metric": f"C5 inference sweep ASTs/s, {mode}, K1 pack + fused forward",
            "unit": "ASTs/s", "by_n": res, "dtype": precision}


def full():
    out = []
    lib = pb._lib.load()
    cfg = pb.full_reference_config()
    p = pb.Predictor(pb.init_params(cfg))
    assert p.large is not None
    big = synth.generate(16384, seed=0)
    flops_ast = None
    for n in (600, 4096, 16384):
        sub = big.take(np.arange(n))
        r = rag(sub)
        rows, ordering, leaf_off, devfeat = engine.upload_ragged(r, torch.device("cuda"))
        f = lambda: p.forward_device(rows, ordering, leaf_off, devfeat, n, False, None,  # noqa
                                     latents=False, n_leaf=r.n_leaf)
        for _ in range(3):
            f()
        t = dev_time(f, 5)
        L = sub.n_leaf.astype(np.float64)
        d, ff, de = cfg.d_model, cfg.d_ff, cfg.d_embed
        fl = (2 * L * 24 * d + cfg.n_layers * (8 * L * d * d + 4 * L * L * d + 4 * L * d * ff)
              + 2 * L * d * de + 2 * 6 * cfg.d_device + 2 * cfg.d_device * de + de)
        dims = [de] + list(cfg.decoder_dims) + [1]
        fl = fl + sum(2 * a * b for a, b in zip(dims[:-1], dims[1:]))
        flops_ast = fl.mean()
        out.append({"metric": f"full_reference_config inference ASTs/s (n={n}, 1 GPU)",
                    "value": n / t, "unit": "ASTs/s", "ms": t * 1e3,
                    "model_tflops": n * flops_ast / t / 1e12,
                    "mflop_per_ast": flops_ast / 1e6,
                    "dtype": "3xTF32 tcgen05 GEMMs, fp32 accumulate"})
    # the GEMM alone (pre-split operands): QKV-shaped, M = 16384 tokens
    import os
    for M, N, K in ((16384, 2148, 736), (16384, 716, 992), (65536, 716, 736)):
        kp = (K + 31) // 32 * 32
        a = [torch.randn(M, kp, device="cuda") for _ in range(2)]
        b = [torch.randn(N, kp, device="cuda") for _ in range(2)]
        ldc = (N + 31) // 32 * 32
        c = torch.empty(M, ldc, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        g = lambda: lib.tpcb_gemm3_presplit(a[0].data_ptr(), a[1].data_ptr(), b[0].data_ptr(),  # noqa
                                            b[1].data_ptr(), M, N, kp, c.data_ptr(), ldc, s)
        for _ in range(3):
            g()
        t = dev_time(g, 20)
        useful = 2.0 * M * N * K
        out.append({"metric": f"gemm3 {M}x{N}x{K} (3xTF32, pre-split)", "ms": t * 1e3,
                    "useful_tflops": useful / t / 1e12,
                    "tensor_pipe_tf32_tflops": 3 * 2.0 * M * N * kp / t / 1e12})
    return out


def fulltrain(n_steps=40):
    """full_reference_config training samples/s (bs 600, the reference's
    batch; C2 data) through the large path: forward + loss + backward +
    Adam + weight-image rebuild per step (the paper's V100 figure for this
    config is 14,241 samples/s)."""
    from paper_2311_09690_b200.large_training import LargeTrainer
    from paper_2311_09690_b200.training import plan_epoch
    cfg = pb.full_reference_config()
    data = synth.generate(65536, seed=0)
    norm = fit_boxcox(data.latency)
    loss = engine.loss_struct("hybrid", cfg.lambda_hybrid, norm.loss_offset)
    tr = LargeTrainer(cfg, pb.init_params(cfg).tensors, rag(data), norm.encode(data.latency), loss)
    flat, steps = plan_epoch(np.random.default_rng(0), tr.n_leaf, cfg.batch_size)
    warm = steps[:3]
    tr.run_epoch(cfg.lr, flat, warm)
    torch.cuda.synchronize()
    sel = steps[3:3 + n_steps]
    n_samples = int(sel[:, 1].sum())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record()
    tr.run_epoch(cfg.lr, flat, sel)
    b.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    t = a.elapsed_time(b) / 1e3
    losses = tr.losses[:len(sel)].cpu().numpy()
    fl = 3 * 281.0e6  # ≈ 3 × forward MFLOP/sample at the synthetic histogram
    return {"metric": "full_reference_config training samples/s (bs 600, 1 GPU)",
            "value": n_samples / t, "unit": "samples/s", "steps": len(sel),
            "ms_per_step": t / len(sel) * 1e3, "wall_samples_per_s": n_samples / wall,
            "model_tflops": n_samples * fl / t / 1e12, "loss_first_last": [float(losses[0]),
                                                                          float(losses[-1])],
            "paper_v100_samples_per_s": 14241,
            "dtype": "3xTF32 tcgen05 GEMMs, fp32 params/Adam"}


def c4dp():
    import os
    import torch.distributed as dist
    from paper_2311_09690_b200.sampling import kmeans_sharded
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    world, rank = dist.get_world_size(), dist.get_rank()
    n, k = 1 << 20, 1024
    data = synth.generate(n, seed=0)
    off = data.offsets()
    pooled = np.add.reduceat(data.vectors.astype(np.float64), off[:-1], axis=0) / data.n_leaf[:, None]
    part = np.array_split(np.arange(n), world)[rank]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = kmeans_sharded(pooled[part], k, seed=0, assign="tc")
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    tt = torch.tensor([t], dtype=torch.float64, device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return {"metric": f"C4 point-sharded KMeans {n}x{k} d24 (k-means++ + Lloyd, tc assign)",
            "n_gpus": world, "seconds": float(tt.item()), "sizes_sum": int(m.sizes.sum())}


if __name__ == "__main__":
    which = sys.argv[1:] or ["c3", "c4", "c4tc", "c5", "c5bf16", "full", "fulltrain", "c4dp"]
    for w in which:
        r = {"c3": c3, "c4": c4, "c4tc": lambda: c4("tc"), "c5": c5,
             "c5bf16": lambda: c5("bf16"), "full": full, "fulltrain": fulltrain,
             "c4dp": c4dp}[w]()
        for line in (r if isinstance(r, list) else [r]):
            print(json.dumps(line), flush=True)
