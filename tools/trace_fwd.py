"""Per-phase cycle trace of the fp32 parity forward (CTA 0, its last 8 tiles).
python tools/trace_fwd.py [n_ast]"""
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
R = int(sys.argv[2]) if len(sys.argv) > 2 else None
p = pb.Predictor(pb.init_params(pb.desk_config(seed=0)), precision="fp32", rows_per_tile=R)
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
if p.R == 128:  # forward_f32.cu (desk fast path)
    names = {1: "x+inproj", 20: "leaf_embed", 21: "head+decoder"}
    for li in range(2):
        for k, nm in enumerate(["qkv", "attn", "wo+ln1", "ffn1", "ffn2+ln2"]):
            names[2 + 6 * li + k] = f"L{li} {nm}"
    end = 21
else:
    names = {1: "x->smem", 2: "inproj", 20: "encoder", 21: "leaf_embed", 22: "dev mlp+gate",
             23: "decoder", 24: "out+decode"}
    for li in range(2):
        for k, nm in enumerate(["qkv", "attn", "wo", "ln1", "ffn1", "ffn2+ln2"]):
            names[3 + 6 * li + k] = f"L{li} {nm}"
    end = 24
for tile in range(8):
    row = b[tile]
    ids = sorted([i for i in range(31) if row[i]], key=lambda i: row[i])
    prev = row[0]
    parts = []
    for i in ids[1:]:
        parts.append(f"{names.get(i, i)}:{row[i] - prev}")
        prev = row[i]
    print(f"tile: total {row[end] - row[0]} cycles | " + ", ".join(parts))
