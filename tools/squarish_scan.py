"""Random roughly-square shapes (1000-9000, dimensions within 25% of each other, any
residue): dgemm0 against cuBLAS and the selected Strassen configuration against both --
correctness (normwise against cuBLAS) and plan anomalies.   usage: squarish_scan.py [n] [seed]"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

n_shapes = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
ctx = S.Ctx()
N = 5


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(N):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / N * 1e-3


worst_err, rows = 0.0, []
for _ in range(n_shapes):
    base = rng.randint(1000, 9000)
    m, n, k = (max(256, int(base * rng.uniform(0.8, 1.25)) + rng.choice([0, 0, 1, 3, 4, 8, -1]))
               for _ in range(3))
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda") * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda") * 2 - 1).t()
    C0 = (torch.rand(n, m, dtype=torch.float64, device="cuda") * 2 - 1).t()
    Cc = C0.t().clone()  # (n, m) contiguous = column-major (m, n): cuBLAS without a copy
    t_cu = timed(lambda: Cc.addmm_(B.t(), A.t()))
    ref = C0 + A @ B
    scale = (A.norm() * B.norm()).item()
    v, L, _ = S.select(m, n, k)
    line = f"{m:5d}x{n:5d}x{k:5d} cublas {2.0 * m * n * k / t_cu / 1e12:5.1f}"
    for vv, ll in (("dgemm", 0), (v, L)):
        C = C0.t().clone().t()
        ctx.gemm_device(vv, ll, 1.0, A, B, C)
        torch.cuda.synchronize()
        err = ((C - ref).norm() / scale).item()
        worst_err = max(worst_err, err)
        assert err <= 5e-12, (m, n, k, vv, ll, err)
        t = timed(lambda: ctx.gemm_device(vv, ll, 1.0, A, B, C))
        line += f" | {vv}{ll} {2.0 * m * n * k / t / 1e12:5.1f} ({t_cu / t:4.2f}x)"
    rows.append(line)
    print(line, flush=True)
    del A, B, C0, Cc, ref, C
print("worst normwise", worst_err)
