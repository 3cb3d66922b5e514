"""Random shapes: the library's configurations against cuBLAS DGEMM (torch addmm_),
back-to-back calls, to find plans that fall off.   usage: random_scan.py [n] [seed] [confs]"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

n_shapes = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
confs = (sys.argv[3] if len(sys.argv) > 3 else "dgemm0").split(",")
ctx = S.Ctx()
N = 8


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(N):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / N * 1e-3


rows = []
for _ in range(n_shapes):
    m, n, k = (rng.choice([1, 8, 16, 64]) * rng.randint(8, 90) for _ in range(3))
    m, n, k = max(m, 64), max(n, 64), max(k, 32)
    if m * n * 8 > 2e9 or m * k * 8 > 2e9 or k * n * 8 > 2e9 or 2.0 * m * n * k < 2e8:
        continue
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda") * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda") * 2 - 1).t()
    C = (torch.rand(n, m, dtype=torch.float64, device="cuda") * 2 - 1).t()
    t_cu = timed(lambda: C.addmm_(A, B))
    out = [f"{m:5d}x{n:5d}x{k:5d} cublas {2.0 * m * n * k / t_cu / 1e12:5.1f} TF/s"]
    worst = 0.0
    for vl in confs:
        v, L = vl[:-1], int(vl[-1])
        t = timed(lambda: ctx.gemm_device(v, L, 1.0, A, B, C))
        out.append(f"{vl} {2.0 * m * n * k / t / 1e12:5.1f} ({t_cu / t:4.2f}x)")
        worst = max(worst, t / t_cu) if vl == "dgemm0" else worst
    rows.append((worst, "  ".join(out)))
    del A, B, C
for w, line in sorted(rows, reverse=True):
    print(line, flush=True)
