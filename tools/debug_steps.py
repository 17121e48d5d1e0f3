import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2311_09690_b200 as pb
from paper_2311_09690_b200 import engine, synth
from paper_2311_09690_b200.dataset import fit_boxcox
from paper_2311_09690_b200.training import Trainer
from oracle import featurize as of, predictor as op, trainer as ot

data = synth.generate(2048, seed=3)
norm = fit_boxcox(data.latency)
y = norm.encode(data.latency)
cfg = pb.desk_config(seed=0)
params = pb.init_params(cfg)
dv = pb.device_vector(pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0))
rag = engine.RaggedHost(rows=data.vectors, ordering=data.ordering, n_leaf=data.n_leaf,
                        devfeat=np.tile(dv, (data.n, 1)).astype(np.float32), encoded=False)
loss = engine.loss_struct("hybrid", 1e-3, norm.loss_offset, 0.0, 5, "transformed", norm)
tr = Trainer(cfg, params.tensors, rag, y, loss, use_graph=False)
flat, steps = tr.plan(np.random.default_rng(0))
NS = 40
T = {k: v.copy() for k, v in params.tensors.items()}
dm = op.Dims(64, 2, 2, 128, 32, 16, (64, 64), 16)
opt = ot.AdamState(T)
off = data.offsets()
for s in range(NS):
    o, n = steps[s][:2]
    b = flat[o:o + n]
    L = int(data.n_leaf[b[0]])
    # device: one step
    tr.run_epoch(1e-3, flat, steps[s:s + 1].copy())
    tr.stream.synchronize()
    got = float(tr.step_loss[0].item())
    x = np.stack([of.encode_rows(data.vectors[off[i]:off[i] + L], data.ordering[off[i]:off[i] + L]) for i in b])
    want = ot.train_step(T, dm, x, np.tile(dv, (n, 1)), y[b], opt, 1e-3, norm.loss_offset)
    dev_T = tr.tensors()
    perr = max(np.abs(dev_T[k] - T[k]).max() / (np.abs(T[k]).max() + 1e-12) for k in T)
    worst = max(T, key=lambda k: np.abs(dev_T[k] - T[k]).max() / (np.abs(T[k]).max() + 1e-12))
    print(f"step {s:3d} L={L} n={n:2d} loss dev {got:.6f} ref {want:.6f} rel {abs(got-want)/abs(want):.2e}  param relerr {perr:.2e} ({worst})")
