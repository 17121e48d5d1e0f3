"""Kernel-time breakdown of one full_reference_config forward (large path)
with the CUPTI activity trace of torch.profiler (device times per kernel
name, summed).  python tools/large_profile.py [n_ast] [precision]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import engine, synth  # noqa: E402
from bench_extra import rag  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
if prec == "train":  # one bs-600 training step (n ignored)
    from paper_2311_09690_b200.dataset import fit_boxcox
    from paper_2311_09690_b200.large_training import LargeTrainer
    from paper_2311_09690_b200.training import plan_epoch
    cfg = pb.full_reference_config()
    data = synth.generate(16384, seed=0)
    norm = fit_boxcox(data.latency)
    loss = engine.loss_struct("hybrid", cfg.lambda_hybrid, norm.loss_offset)
    tr = LargeTrainer(cfg, pb.init_params(cfg).tensors, rag(data), norm.encode(data.latency),
                      loss)
    flat, steps = plan_epoch(np.random.default_rng(0), tr.n_leaf, cfg.batch_size)
    big = steps[steps[:, 1] == cfg.batch_size][:1]
    f = lambda: tr.run_epoch(cfg.lr, flat, big)  # noqa
else:
    p = pb.Predictor(pb.init_params(pb.full_reference_config()), precision=prec)
    sub = synth.generate(n, seed=0)
    r = rag(sub)
    rows, ordering, leaf_off, devfeat = engine.upload_ragged(r, torch.device("cuda"))
    f = lambda: p.forward_device(rows, ordering, leaf_off, devfeat, n, False, None,  # noqa
                                 latents=False, n_leaf=r.n_leaf)
for _ in range(3):
    f()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    f()
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        full = e.name
        name = full[:90]
        for key in ("gemm3_kernel<128>", "gemm3_kernel<256>", "attention_back_kernel",
                    "attention_kernel", "layernorm_kernel", "ln_back_kernel", "transpose_pair",
                    "colsum_kernel", "reduce_grad", "build_image", "optimizer_kernel",
                    "device_gate", "gate_back", "out_back", "output_kernel", "gather_tokens",
                    "loss_kernel", "featurize", "pack"):
            if key in full:
                name = key
                break
        if name.startswith("gemm3") and e.input_shapes is not None:
            pass
        t, c = agg.get(name, (0.0, 0))
        agg[name] = (t + e.device_time_total, c + 1)
tot = sum(t for t, _ in agg.values())
for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{t / 1e3:9.3f} ms  {100 * t / tot:5.1f} %  x{c:4d}  {k[:90]}")
print(f"{tot / 1e3:9.3f} ms total kernel time, n={n}")
