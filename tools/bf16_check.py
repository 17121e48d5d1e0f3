"""bf16 tensor-core forward vs the fp32 parity path: accuracy (desk trained
checkpoint, C1 set) and throughput sweep.  python tools/bf16_check.py"""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from conftest import GoldenModel, load_golden  # noqa: E402
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import engine, synth  # noqa: E402
from oracle import featurize as of  # noqa: E402

gm = GoldenModel("desk")
params = pb.CostModelParams(pb.CostModelConfig(**gm.cfg), gm.T)
c1 = load_golden("c1_4096")
lam, sh, tm, ts, loff = gm.z["norm"]
norm = pb.BoxCoxNormalizer(lam, sh, True, tm, ts, loff)
dv = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0).astype(np.float32)
n = len(c1["n_leaf"])
rag = engine.RaggedHost(rows=c1["vectors"].astype(np.float32), ordering=c1["ordering"],
                        n_leaf=c1["n_leaf"], devfeat=np.tile(dv, (n, 1)), encoded=False)
out = {}
for prec in ("fp32", "bf16"):
    p = pb.Predictor(params, precision=prec)
    pred, zx, zv, z, lat = p.forward_ragged(rag, norm, latents=True)
    out[prec] = (pred.cpu().numpy(), lat.cpu().numpy(), zx.cpu().numpy())
d_pred = np.abs(out["bf16"][0] - out["fp32"][0])
rel_lat = np.abs(out["bf16"][1] - out["fp32"][1]) / np.abs(out["fp32"][1])
print(f"model-space pred: max |d| {d_pred.max():.3e}  mean {d_pred.mean():.3e}")
print(f"decoded latency rel err: max {rel_lat.max():.3e}  mean {rel_lat.mean():.3e}  p99 {np.quantile(rel_lat, 0.99):.3e}")
print(f"z_x max |d| {np.abs(out['bf16'][2] - out['fp32'][2]).max():.3e}")
big = synth.generate(1 << 20, seed=0)
for prec in ("fp32", "bf16"):
    p = pb.Predictor(pb.init_params(pb.desk_config(seed=0)), precision=prec)
    res = {}
    for m in (4096, 65536, 1 << 20):
        sub = big.take(np.arange(m))
        r = engine.RaggedHost(rows=sub.vectors.astype(np.float32), ordering=sub.ordering,
                              n_leaf=sub.n_leaf, devfeat=np.tile(dv, (m, 1)), encoded=False)
        rows, ordering, leaf_off, devfeat = engine.upload_ragged(r, torch.device("cuda"))
        f = lambda: p.forward_device(rows, ordering, leaf_off, devfeat, m, False, None, latents=False)  # noqa
        for _ in range(3):
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        reps = 20 if m <= 65536 else 5
        for _ in range(reps):
            f()
        b.record()
        torch.cuda.synchronize()
        res[m] = m * reps / (a.elapsed_time(b) / 1e3)
    print(prec, {k: f"{v/1e6:.1f}M" for k, v in res.items()})
