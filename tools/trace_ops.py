"""(kernel selection / grid cap: TPCB_TRAIN_IMPL / TPCB_GRID_CAP env vars)
Per-op cycle trace of CTA 0 (v3/v4 kernels): wait for weights vs work.
python tools/trace3.py [impl=4]"""
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
impl = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tr = Trainer(cfg, pb.init_params(cfg).tensors, rag, y, loss, use_graph=False)
flat, steps = tr.plan(np.random.default_rng(0))
tr.run_epoch(1e-3, flat, steps[:3].copy())
tr.stream.synchronize()
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
lib = _lib.load()
Ls = [int(a) for a in sys.argv[2:]] or [5]
cap = int(__import__('os').environ.get('GRID_CAP', '0'))
step_L = data.n_leaf[flat[steps[:, 0]]]
for want in Ls:
    cand = np.nonzero(step_L == want)[0]
    if not len(cand):
        print("no step with L", want)
        continue
    si = int(cand[0])
    lib.tpcb_debug_train_trace(buf.data_ptr())
    buf.zero_()
    tr.run_epoch(1e-3, flat, steps[si:si + 1].copy())
    tr.stream.synchronize()
    lib.tpcb_debug_train_trace(None)
    raw = buf.cpu().numpy()
    b = raw[:256].reshape(-1, 2)
    n = int(np.count_nonzero(b[:, 0]))
    t0, t1 = int(raw[510]), int(raw[511])
    ph = raw[256:510]
    ids = [i for i in range(254) if ph[i]]
    if ids:
        prev = t0
        out = []
        for i in ids:
            out.append(f"{i}:{int(ph[i] - prev)}")
            prev = ph[i]
        print("  phases (id:cycles since previous mark)", " ".join(out))
    print(f"L={want} (step {si}, n={steps[si][1]}) slots={n} sample span={t1 - t0} cycles "
          f"({(t1 - t0) / 1965:.1f} us @1.965 GHz)")
    tw = tk = 0
    row = []
    for i in range(n):
        wait = b[i, 1] - b[i, 0]
        work = (b[i + 1, 0] - b[i, 1]) if i + 1 < n else t1 - b[i, 1]
        tw += wait; tk += work
        row.append(f"{i}:{wait}/{work}")
    print("  pre", b[0, 0] - t0, " slot:wait/work", " ".join(row))
    print("  wait sum", tw, "work sum", tk)
