"""Per-op cycle trace of CTA 0 of the training kernel for one step."""
import ctypes as C
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
if len(sys.argv) > 1:  # fewer gradient slots → several samples per CTA
    tr.ws = engine.TrainWorkspace(tr.dm, int(sys.argv[1]))
flat, steps = tr.plan(np.random.default_rng(0))
tr.run_epoch(1e-3, flat, steps[:3].copy())
tr.stream.synchronize()
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.tpcb_debug_train_trace(buf.data_ptr())
for k in range(3, 8):
    buf.zero_()
    tr.run_epoch(1e-3, flat, steps[k:k + 1].copy())
    tr.stream.synchronize()
    for rep in (0, 1):
        b4 = buf.cpu().numpy()[256 * rep:256 * rep + 256].reshape(-1, 4)
        b = b4[:, [0, 3]]
        n = int(np.count_nonzero(b[:, 0]))
        if n == 0:
            continue
        L = int(data.n_leaf[flat[steps[k][0]]])
        t0 = b[0, 0]
        rows = []
        for i in range(n):
            wait = b[i, 1] - b[i, 0]
            work = (b[i + 1, 0] - b[i, 1]) if i + 1 < n else 0
            rows.append((i, wait, work))
        tot = b[n - 1, 1] - t0
        print(f"rep {rep} step {k} L={L}: {n} ops, span {tot} cycles ({tot/1.965e3:.1f} us); wait sum {sum(r[1] for r in rows)}, work sum {sum(r[2] for r in rows)}")
        if k == 3 and rep == 0:
            for i, r in enumerate(rows):
                print("   op %2d  wait %6d  work %6d   (issue %5d, cp.async wait %5d, barrier %5d)"
                      % (r + (b4[i, 1] - b4[i, 0], b4[i, 2] - b4[i, 1], b4[i, 3] - b4[i, 2])))
lib.tpcb_debug_train_trace(None)
