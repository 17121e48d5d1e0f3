import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2311_09690_b200 as pb
from paper_2311_09690_b200 import engine, synth
from paper_2311_09690_b200.costmodel import LossSpec, backward
from paper_2311_09690_b200.dataset import fit_boxcox
from paper_2311_09690_b200.training import epoch_batches
from oracle import featurize as of, predictor as op, trainer as ot

data = synth.generate(2048, seed=3)
norm = fit_boxcox(data.latency)
y = norm.encode(data.latency)
cfg = pb.desk_config(seed=0)
params = pb.init_params(cfg)
dv = pb.device_vector(pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0))
T = {k: v.copy() for k, v in params.tensors.items()}
dm = op.Dims(64, 2, 2, 128, 32, 16, (64, 64), 16)
opt = ot.AdamState(T)
off = data.offsets()
batches = epoch_batches(np.random.default_rng(0), data.n_leaf, 64)
for s in range(6):
    b = batches[s]
    L = int(data.n_leaf[b[0]])
    x = np.stack([of.encode_rows(data.vectors[off[i]:off[i] + L], data.ordering[off[i]:off[i] + L]) for i in b])
    dev = np.tile(dv, (len(b), 1))
    pred, _, _, _, tape = op.bucket_forward(T, dm, x, dev)
    val, dpred = op.loss_and_grad(pred, y[b], "hybrid", 1e-3, norm.loss_offset)
    G = {}
    op.bucket_backward(T, dm, tape, dpred, None, G)
    inputs = [pb.EncodedInput(x[i], dev[i]) for i in range(len(b))]
    v2, g2, aux = backward(pb.CostModelParams(cfg, T), inputs, y[b],
                           LossSpec(mode="hybrid", lambda_hybrid=1e-3, offset=norm.loss_offset))
    print(f"step {s} L={L} loss {val:.6f} dev {v2:.6f}")
    for k in T:
        ref = G.get(k, np.zeros_like(T[k]))
        got = g2[k]
        mx = np.abs(ref).max()
        if mx == 0: continue
        err = np.abs(got - ref).max() / mx
        sig = np.abs(ref) > 1e-4 * mx
        flips = int(np.sum(np.sign(got[sig]) != np.sign(ref[sig])))
        if err > 1e-4 or flips:
            i = np.unravel_index(np.argmax(np.abs(got - ref)), ref.shape)
            print(f"   {k:22s} err {err:.2e} flips {flips} max|g| {mx:.2e} worst at {i}: ref {ref[i]:.4e} got {got[i]:.4e}")
    opt.step(T, G, 1e-3)
