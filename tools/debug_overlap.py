"""A/B one training step: sequential reduce vs overlapped reduce."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import paper_2311_09690_b200 as pb
from paper_2311_09690_b200 import _lib
from paper_2311_09690_b200.training import Trainer
from test_gpu_training_loop import _oracle_setup

data, norm, y, dv, rag, loss = _oracle_setup(n=2048)
cfg = pb.desk_config(seed=0)
params = pb.init_params(cfg)
lib = _lib.load()
nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
res = []
for on in (0, 1):
    lib.tpcb_debug_overlap(on)
    tr = Trainer(cfg, params.tensors, rag, y, loss, use_graph=False)
    flat, steps = tr.plan(np.random.default_rng(3))
    tr.run_epoch(1e-3, flat, steps[:nsteps].copy())
    tr.stream.synchronize()
    res.append((tr.step_loss[:nsteps].cpu().numpy(), tr.tensors(), int(tr.status.t.item()),
                tr.m.cpu().numpy(), tr.v.cpu().numpy()))
    print("overlap", on, "status", res[-1][2], "losses", res[-1][0])
a, b = res
for k in a[1]:
    d = np.abs(a[1][k] - b[1][k]).max()
    if d > 0:
        print(f"{k:22s} maxdiff {d:.3e}")
print("m diff", np.abs(a[3] - b[3]).max(), "v diff", np.abs(a[4] - b[4]).max())
