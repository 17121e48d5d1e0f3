"""Per-op cycle trace of CTA 0 (v3 kernel): wait for weights vs work."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2311_09690_b200 as pb
from paper_2311_09690_b200 import _lib, engine, synth
from paper_2311_09690_b200.dataset import fit_boxcox
from paper_2311_09690_b200.training import Trainer

data = synth.generate(4096, seed=0)
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
tr.run_epoch(1e-3, flat, steps[:3].copy())
tr.stream.synchronize()
buf = torch.zeros(256, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.tpcb_debug_train_trace(buf.data_ptr())
buf.zero_()
tr.run_epoch(1e-3, flat, steps[3:4].copy())
tr.stream.synchronize()
lib.tpcb_debug_train_trace(None)
b = buf.cpu().numpy().reshape(-1, 2)
n = int(np.count_nonzero(b[:, 0]))
L = int(data.n_leaf[flat[steps[3][0]]])
print(f"L={L} ops={n} span={b[n-1,1]-b[0,0]} cycles ({(b[n-1,1]-b[0,0])/1965:.1f} us)")
tw = tk = 0
for i in range(n):
    wait = b[i, 1] - b[i, 0]
    work = (b[i + 1, 0] - b[i, 1]) if i + 1 < n else 0
    tw += wait; tk += work
    print("op %2d wait %6d work %6d" % (i, wait, work))
print("wait sum", tw, "work sum", tk)
