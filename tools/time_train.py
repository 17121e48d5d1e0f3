"""(kernel selection / grid cap: TPCB_TRAIN_IMPL / TPCB_GRID_CAP env vars)
Quick per-step timing of the training epoch (profiled + graph), desk config.
python tools/time_train.py [n_samples]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import engine, synth  # noqa: E402
from paper_2311_09690_b200.dataset import fit_boxcox  # noqa: E402
from paper_2311_09690_b200.training import Trainer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
impl = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # 0 auto, 2 generic, 3, 4 fast path
from paper_2311_09690_b200 import _lib  # noqa: E402
data = synth.generate(n, seed=0)
norm = fit_boxcox(data.latency)
y = norm.encode(data.latency)
cfg = pb.desk_config(seed=0)
dv = pb.device_vector(pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0))
rag = engine.RaggedHost(rows=data.vectors.astype(np.float32), ordering=data.ordering,
                        n_leaf=data.n_leaf, devfeat=np.tile(dv, (data.n, 1)).astype(np.float32),
                        encoded=False)
loss = engine.loss_struct("hybrid", 1e-3, norm.loss_offset, 0.0, 5, "transformed", norm)
tr = Trainer(cfg, pb.init_params(cfg).tensors, rag, y, loss)
rng = np.random.default_rng(0)
flat, steps = tr.plan(rng)
ns = steps.shape[0]
prof = np.zeros(3)
tr.run_epoch(1e-3, flat, steps, profile=prof)
print(f"steps/epoch {ns}: per step  train {prof[0]/ns*1e3:.1f} us  reduce+adam {prof[1]/ns*1e3:.1f} us")
for rep in range(3):
    flat, steps = tr.plan(rng)
    tr.stream.synchronize()
    t0 = time.perf_counter()
    tr.run_epoch(1e-3, flat, steps)
    tr.stream.synchronize()
    dt = time.perf_counter() - t0
    print(f"graph epoch: {dt*1e3:.1f} ms  -> {dt/ns*1e6:.1f} us/step, {n*0.8/dt:.0f} samples/s")
print("last losses", tr.step_loss[:ns].cpu().numpy()[-3:])
