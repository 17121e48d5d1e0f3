"""One full_reference_config training step (bs 600) through the large path,
for ncu launch lists: python tools/large_step.py [warmup_steps]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import engine, synth  # noqa: E402
from paper_2311_09690_b200.dataset import fit_boxcox  # noqa: E402
from paper_2311_09690_b200.large_training import LargeTrainer  # noqa: E402
from paper_2311_09690_b200.training import plan_epoch  # noqa: E402

cfg = pb.full_reference_config()
data = synth.generate(16384, seed=0)
norm = fit_boxcox(data.latency)
loss = engine.loss_struct("hybrid", cfg.lambda_hybrid, norm.loss_offset)
dv = pb.device_vector(pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0))
rag = engine.RaggedHost(rows=data.vectors.astype(np.float32), ordering=data.ordering,
                        n_leaf=data.n_leaf, devfeat=np.tile(dv, (data.n, 1)).astype(np.float32),
                        encoded=False)
tr = LargeTrainer(cfg, pb.init_params(cfg).tensors, rag, norm.encode(data.latency), loss)
flat, steps = plan_epoch(np.random.default_rng(0), tr.n_leaf, cfg.batch_size)
big = steps[steps[:, 1] == cfg.batch_size]
L_of = [int(tr.n_leaf[flat[s[0]]]) for s in big]
pick = big[[L_of.index(4)]]  # a bs-600 step of leaf count 4 (the mean is 3.6)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    tr.run_epoch(cfg.lr, flat, pick)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
tr.run_epoch(cfg.lr, flat, pick)
b.record()
torch.cuda.synchronize()
print(f"step ms {a.elapsed_time(b):.3f}")
