"""One pre-split 3xTF32 tcgen05 GEMM launch (for ncu):
python tools/gemm_probe.py [M N K] [reps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2311_09690_b200 import _lib  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (16384, 2148, 736)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
lib = _lib.load()
kp = (K + 31) // 32 * 32
a = [torch.randn(M, kp, device="cuda") for _ in range(2)]
b = [torch.randn(N, kp, device="cuda") for _ in range(2)]
ldc = (N + 31) // 32 * 32
c = torch.empty(M, ldc, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    _lib.check(lib.tpcb_gemm3_presplit(a[0].data_ptr(), a[1].data_ptr(), b[0].data_ptr(),
                                       b[1].data_ptr(), M, N, kp, c.data_ptr(), ldc, s), "gemm3")
torch.cuda.synchronize()
print("ok")
