"""Randomised stress run through the C ABI: random shapes (including ragged and
degenerate ones), layouts (column-/row-major, C inside a larger buffer), alphas,
variants and levels (level 3 included), host and device pointers; every result is
checked against cuBLAS (normwise, BASELINE tolerances) and nothing outside C may
change.  usage: python tools/stress.py [seconds=240] [seed=0]"""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1605_01078_b200 as S

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
ctx = S.Ctx()
ctx.set_max_level(3)
CFG = [("dgemm", 0), ("abc", 1), ("ab", 1), ("naive", 1), ("c", 1), ("abc", 2), ("ab", 2),
       ("naive", 2), ("c", 2), ("naive", 3), ("c", 3)]
TOL = {0: 1e-12, 1: 1e-12, 2: 5e-12, 3: 2e-11}
t_end = time.time() + budget
n_runs = worst = 0
fails = []
while time.time() < t_end:
    big = rng.random() < 0.25
    hi = 5000 if big else 900
    m, n, k = (rng.choice([rng.randint(1, hi), rng.randint(1, 64), rng.randrange(128, hi + 1, 128)])
               for _ in range(3))
    v, L = rng.choice(CFG)
    alpha = rng.choice([1.0, -1.0, 0.5, 2.0])
    g = torch.Generator(device="cuda").manual_seed(rng.randrange(1 << 30))
    A = torch.rand(m, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B = torch.rand(k, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    if rng.random() < 0.5:
        A = A.t().contiguous().t()  # column-major
    if rng.random() < 0.5:
        B = B.t().contiguous().t()
    pad_r, pad_c = rng.choice([0, 0, 3, 8]), rng.choice([0, 0, 2])
    colmajor = rng.random() < 0.7
    if colmajor:
        buf = torch.full((n + pad_c, m + pad_r), -777.25, dtype=torch.float64, device="cuda").t()
    else:
        buf = torch.full((m + pad_r, n + pad_c), -777.25, dtype=torch.float64, device="cuda")
    C = buf[:m, :n]
    C.copy_(torch.rand(m, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
    want = C + alpha * (A @ B)
    host = rng.random() < 0.3
    if host:
        Ah, Bh = A.cpu(), B.cpu()
        bh = buf.cpu()
        Ch = bh[:m, :n]
        ctx.gemm(v, L, alpha, Ah, Bh, Ch)
        buf.copy_(bh)
    else:
        ctx.gemm_device(v, L, alpha, A, B, C)
    torch.cuda.synchronize()
    outside = buf.clone()
    outside[:m, :n] = -777.25
    den = (torch.linalg.norm(A) * torch.linalg.norm(B)).item() or 1.0
    nw = (torch.linalg.norm(C - want) / den).item()
    n_runs += 1
    worst = max(worst, nw)
    ok = nw <= TOL[L] and bool((outside == -777.25).all())
    if not ok:
        fails.append((m, n, k, v, L, alpha, host, colmajor, pad_r, pad_c, nw))
        print("FAIL", fails[-1], flush=True)
print(f"stress: {n_runs} calls, worst normwise {worst:.2e}, failures {len(fails)}", flush=True)
sys.exit(1 if fails else 0)
