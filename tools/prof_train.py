"""Run a few training steps (no graph) — target for ncu captures of the
train-step kernels.  python tools/prof_train.py [n_steps]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import engine, synth  # noqa: E402
from paper_2311_09690_b200.dataset import fit_boxcox  # noqa: E402
from paper_2311_09690_b200.training import Trainer  # noqa: E402

n_steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
data = synth.generate(16384, seed=0)
norm = fit_boxcox(data.latency)
y = norm.encode(data.latency)
cfg = pb.desk_config(seed=0)
dv = pb.device_vector(pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0))
rag = engine.RaggedHost(rows=data.vectors.astype(np.float32), ordering=data.ordering,
                        n_leaf=data.n_leaf, devfeat=np.tile(dv, (data.n, 1)).astype(np.float32),
                        encoded=False)
loss = engine.loss_struct("hybrid", 1e-3, norm.loss_offset, 0.0, 5, "transformed", norm)
tr = Trainer(cfg, pb.init_params(cfg).tensors, rag, y, loss, use_graph=False)
flat, steps = tr.plan(np.random.default_rng(0))
tr.run_epoch(1e-3, flat, steps[:n_steps])
tr.stream.synchronize()
print("ok", tr.step_loss[:n_steps].cpu().numpy()[:4])
