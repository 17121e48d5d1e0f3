import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2311_09690_b200 import sampling as s
rng = np.random.default_rng(3)
x = np.concatenate([rng.normal(loc=rng.normal(scale=4, size=32), size=(512, 32)) for _ in range(8)])
for k in (256, 257, 300, 512, 1024):
    init = x[rng.choice(len(x), k, replace=False)]
    ex = s.DeviceKMeans(x, k); tc = s.DeviceKMeans(x, k, assign="tc")
    for km in (ex, tc):
        km.centers.copy_(torch.from_numpy(init)); km.assign_step()
    a, b = ex.assign.cpu().numpy(), tc.assign.cpu().numpy()
    bad = np.flatnonzero(a != b)
    print(k, "agree", np.mean(a == b), "first bad", bad[:5], a[bad[:5]], b[bad[:5]])
