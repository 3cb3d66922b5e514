"""Host-side cost of one strassen_gemm_device call at small sizes: wall time of
N back-to-back submissions (GPU kept busy) vs the GPU time per call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1605_01078_b200 as S

ctx = S.Ctx()
for d in (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,2048").split(",")):
    A, B, C = ((torch.rand(d, d, dtype=torch.float64, device="cuda") * 2 - 1).t() for _ in range(3))
    for v, L in (("dgemm", 0), ("abc", 1), ("abc", 2), ("naive", 2), ("c", 2)):
        for _ in range(5):
            ctx.gemm_device(v, L, 1.0, A, B, C)
        torch.cuda.synchronize()
        n = 50
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(n):
            ctx.gemm_device(v, L, 1.0, A, B, C)
        e1.record()
        t_host = (time.perf_counter() - t0) / n
        torch.cuda.synchronize()
        t_gpu = e0.elapsed_time(e1) / n * 1e-3
        ctx.enable_profiling(True)
        ctx.gemm_device(v, L, 1.0, A, B, C)
        torch.cuda.synchronize()
        kern = sum(p["ms"] for p in ctx.last_profile()) * 1e-3
        ctx.enable_profiling(False)
        print(f"{d} {v}{L}: host submit {t_host * 1e6:7.1f} us/call  stream time {t_gpu * 1e6:7.1f} us/call"
              f"  kernels {kern * 1e6:7.1f} us  launches {ctx.last_launches()}", flush=True)
