"""Per-phase cycle trace of the bf16 tensor-core forward (CTA 0, first 8 tiles).
python tools/trace_tc.py [n_ast]"""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import _lib, engine, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
data = synth.generate(n, seed=0)
dv = pb.device_vector(pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)).astype(np.float32)
rag = engine.RaggedHost(rows=data.vectors.astype(np.float32), ordering=data.ordering,
                        n_leaf=data.n_leaf, devfeat=np.tile(dv, (n, 1)), encoded=False)
p = pb.Predictor(pb.init_params(pb.desk_config(seed=0)), precision="bf16")
rows, ordering, leaf_off, devfeat = engine.upload_ragged(rag, torch.device("cuda"))
f = lambda: p.forward_device(rows, ordering, leaf_off, devfeat, n, False, None, latents=False)  # noqa
f()
torch.cuda.synchronize()
buf = torch.zeros(256, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.tpcb_debug_train_trace(buf.data_ptr())
f()
torch.cuda.synchronize()
lib.tpcb_debug_train_trace(None)
b = buf.cpu().numpy().reshape(8, 32)
names = {0: "start", 1: "x->A", 2: "inproj mma", 3: "inproj epi"}
for li in range(2):
    base = 4 + 12 * li
    for k, nm in enumerate(["qkv mma", "qkv epi+attn", "wo mma", "ln1 epi", "ffn1 mma", "ffn1 epi",
                            "ffn2 mma", "ln2 epi"]):
        names[base + k] = f"L{li} {nm}"
names[12] = "leaf sync"
names[13] = "leaf B wait"
names[14] = "leaf mma issue"
names[25] = "leaf mma wait"
names[26] = "zx+dev mlp+gate->A"
names[27] = "dec0 mma"
names[28] = "dec0 epi+dec1 mma"
names[30] = "enc done"
names[31] = "dec1 epi+store"
for tile in range(8):
    row = b[tile]
    ids = sorted([i for i in range(32) if row[i]], key=lambda i: row[i])
    prev = row[0]
    parts = []
    for i in ids[1:]:
        parts.append(f"{names.get(i, i)}:{row[i] - prev}")
        prev = row[i]
    print(f"tile {tile}: total {row[31] - row[0]} cycles | " + ", ".join(parts))
