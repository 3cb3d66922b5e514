"""Fixed per-call / per-CTA overhead of the mm launches: back-to-back time per call of
one configuration at fixed m = n while k grows (intercept = the overhead, slope = the
k-step rate).   overhead_probe.py [dgemm0,abc1] [1536,1024,1000] [16,64,256,1024]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

confs = (sys.argv[1] if len(sys.argv) > 1 else "dgemm0,abc1").split(",")
dims = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1536,1024,1000").split(",")]
ks = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "16,64,256,512,1024,1536").split(",")]
N = 30
ctx = S.Ctx()
for d in dims:
    for k in ks:
        A = (torch.rand(k, d, dtype=torch.float64, device="cuda") * 2 - 1).t()
        B = (torch.rand(d, k, dtype=torch.float64, device="cuda") * 2 - 1).t()
        C = (torch.rand(d, d, dtype=torch.float64, device="cuda") * 2 - 1).t()
        line = [f"{d}x{d}x{k}"]
        for vl in confs:
            v, L = vl[:-1], int(vl[-1])
            for _ in range(3):
                ctx.gemm_device(v, L, 1.0, A, B, C)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(N):
                ctx.gemm_device(v, L, 1.0, A, B, C)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / N * 1e3
            ctx.enable_profiling(True)
            ctx.gemm_device(v, L, 1.0, A, B, C)
            torch.cuda.synchronize()
            mm = sum(p["ms"] for p in ctx.last_profile() if p["kernel"] == "mm_kernel") * 1e3
            ctx.enable_profiling(False)
            line.append(f"{vl} {us:7.1f} us (mm {mm:6.1f}, {2.0 * d * d * k / us / 1e6:5.1f} TF/s)")
        print("  ".join(line), flush=True)
