"""Deterministic small cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every variant and level, ragged and tile-multiple shapes, the split
(few-tile), persistent and stream-K launch modes, strided views, device and host
pointers (the host window pipeline).  Each result is checked against cuBLAS.
usage: compute-sanitizer --tool T --error-exitcode 9 python tools/sanitize_cases.py [quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1605_01078_b200 as S

CFG = [("dgemm", 0), ("abc", 1), ("ab", 1), ("naive", 1), ("c", 1), ("abc", 2), ("ab", 2),
       ("naive", 2), ("c", 2), ("naive", 3), ("c", 3)]
TOL = {0: 1e-12, 1: 1e-12, 2: 5e-12, 3: 2e-11}
quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
SHAPES = [(300, 290, 520), (256, 256, 256)] + ([] if quick else [(1000, 1000, 1000),
                                                                 (2048, 2048, 2048)])
ctx = S.Ctx()
ctx.set_max_level(3)
g = torch.Generator(device="cuda").manual_seed(0)
worst, n = 0.0, 0
for (m, nn, k) in SHAPES:
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(nn, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(nn + 3, m + 5, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    want_full = C0.clone()
    want_full[2:2 + m, 1:1 + nn] += A @ B
    scale = (torch.linalg.norm(A) * torch.linalg.norm(B)).item()
    for v, L in CFG:
        for host in (False, True):
            if host and (m, nn, k) == (2048, 2048, 2048) and L == 3:
                continue
            Cf = C0.clone()
            if host:
                Ah, Bh = (x.t().cpu().pin_memory().t() for x in (A, B))
                Ch = Cf.t().cpu().pin_memory().t()
                ctx.gemm(v, L, 1.0, Ah, Bh, Ch[2:2 + m, 1:1 + nn])
                Cf = Ch.cuda()
            else:
                ctx.gemm_device(v, L, 1.0, A, B, Cf[2:2 + m, 1:1 + nn])
                torch.cuda.synchronize()
            err = (torch.linalg.norm(Cf - want_full) / scale).item()
            outside = Cf.clone()
            outside[2:2 + m, 1:1 + nn] = want_full[2:2 + m, 1:1 + nn]
            assert torch.equal(outside, want_full), ("write outside C", v, L, m, nn, k, host)
            assert err <= TOL[L], (v, L, m, nn, k, host, err)
            worst, n = max(worst, err), n + 1
print(f"sanitize cases OK: {n} calls, worst normwise {worst:.2e}")
