"""One shape, one configuration: back-to-back time and the per-launch profile.
usage: shape_ab.py variant level m n k"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

v, L, m, n, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
A = (torch.rand(k, m, dtype=torch.float64, device="cuda") * 2 - 1).t()
B = (torch.rand(n, k, dtype=torch.float64, device="cuda") * 2 - 1).t()
C = (torch.rand(n, m, dtype=torch.float64, device="cuda") * 2 - 1).t()
ctx = S.Ctx()
for _ in range(3):
    ctx.gemm_device(v, L, 1.0, A, B, C)
torch.cuda.synchronize()
N = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N):
    ctx.gemm_device(v, L, 1.0, A, B, C)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / N * 1e-3
e0.record()
for _ in range(N):
    C.addmm_(A, B)
e1.record()
torch.cuda.synchronize()
tc = e0.elapsed_time(e1) / N * 1e-3
ctx.enable_profiling(True)
ctx.gemm_device(v, L, 1.0, A, B, C)
torch.cuda.synchronize()
prof = ctx.last_profile()
print(f"{v}{L} {m}x{n}x{k}: {t * 1e6:8.1f} us {2.0 * m * n * k / t / 1e12:5.1f} TF/s | cublas "
      f"{tc * 1e6:8.1f} us | launches {[(p['kernel'][:8], round(p['ms'] * 1e3, 1)) for p in prof]}")
