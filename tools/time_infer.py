"""Device time of the batched forward (fp32 parity kernel and bf16 tensor-core
kernel) at n ASTs, CUDA events on the launching stream, median of reps.
python tools/time_infer.py [n_ast] [reps]"""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import engine, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
data = synth.generate(n, seed=0)
dv = pb.device_vector(pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)).astype(np.float32)
rag = engine.RaggedHost(rows=data.vectors.astype(np.float32), ordering=data.ordering,
                        n_leaf=data.n_leaf, devfeat=np.tile(dv, (n, 1)), encoded=False)
rows, ordering, leaf_off, devfeat = engine.upload_ragged(rag, torch.device("cuda"))
for prec in ("fp32", "bf16"):
    p = pb.Predictor(pb.init_params(pb.desk_config(seed=0)), precision=prec)
    f = lambda: p.forward_device(rows, ordering, leaf_off, devfeat, n, False, None, latents=False)  # noqa
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    print(f"{prec}: n={n} median {ms:.3f} ms  {n / ms / 1e3:.2f} M ASTs/s")
