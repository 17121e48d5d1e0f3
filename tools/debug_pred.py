"""Compare train-kernel predictions (impl 2 vs 4) on the desk golden batch.
python tools/debug_pred.py"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from conftest import GoldenModel, load_golden  # noqa: E402
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import _lib  # noqa: E402
from paper_2311_09690_b200.costmodel import LossSpec, backward  # noqa: E402
from oracle import featurize as of  # noqa: E402

gm = GoldenModel("desk")
params = pb.CostModelParams(pb.CostModelConfig(**gm.cfg), gm.T)
c1 = load_golden("c1_4096")
off = np.concatenate([[0], np.cumsum(c1["n_leaf"])])
dv = of.device_features(1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
idx = list(gm.z["batch_idx"])
# a mixed batch: the golden batch plus samples of other leaf counts
for L in range(1, 17):
    cand = np.nonzero(c1["n_leaf"] == L)[0]
    idx += list(cand[:2])
batch = [pb.EncodedInput(of.encode_rows(c1["vectors"][off[i]:off[i + 1]],
                                        c1["ordering"][off[i]:off[i + 1]]), dv) for i in idx]
y = np.ones(len(idx))
spec = LossSpec(mode="hybrid", lambda_hybrid=1e-3, offset=1.0)
res = {}
for impl in (2, 4):
    _lib.load().tpcb_debug_train_impl(impl)
    val, grads, aux = backward(params, batch, y, spec)
    res[impl] = (val, grads, aux["pred"])
p2, p4 = res[2][2], res[4][2]
nl = c1["n_leaf"][idx]
print("loss v2", res[2][0], "v4", res[4][0])
for L in sorted(set(nl)):
    m = nl == L
    print(f"L={L:2d} n={m.sum():3d} max|dpred| {np.abs(p2[m] - p4[m]).max():.3e}")
for k in res[2][1]:
    a, b = res[2][1][k], res[4][1][k]
    d = np.abs(a - b).max() / (np.abs(a).max() + 1e-30)
    if d > 1e-3:
        print("grad", k, f"rel {d:.3e}")
