import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2311_09690_b200 as pb
from paper_2311_09690_b200.costmodel import LossSpec, backward
from oracle import predictor as op

cfg = pb.desk_config(seed=0)
T = pb.init_params(cfg).tensors
rng = np.random.default_rng(1)
for k in T:  # non-trivial biases / gains
    T[k] = T[k] + 0.05 * rng.normal(size=T[k].shape)
dm = op.Dims(64, 2, 2, 128, 32, 16, (64, 64), 16)
for L, n in ((1, 1), (1, 3), (2, 1), (1, 64), (3, 64)):
    x = rng.normal(size=(n, L, 24)) * 3
    dev = rng.normal(size=(n, 6))
    y = rng.uniform(1, 3, size=n)
    pred, _, _, _, tape = op.bucket_forward(T, dm, x, dev)
    val, dpred = op.loss_and_grad(pred, y, "mse")
    G = {}
    op.bucket_backward(T, dm, tape, dpred, None, G)
    v2, g2, aux = backward(pb.CostModelParams(cfg, T), [pb.EncodedInput(x[i], dev[i]) for i in range(n)], y, LossSpec(mode="mse"))
    worst = sorted(((np.abs(g2[k] - G[k]).max() / (np.abs(G[k]).max() + 1e-30), k) for k in G), reverse=True)[:4]
    print(f"L={L} n={n} loss {val:.6f} {v2:.6f} pred err {np.abs(aux['pred']-pred).max():.2e} worst", [(f"{e:.1e}", k) for e, k in worst])
