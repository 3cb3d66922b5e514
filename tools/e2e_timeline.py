"""Kernel timeline of one host-pointer strassen_gemm call (profiling on): where the
end-to-end time goes beyond the kernels.  usage: e2e_timeline.py [dim] [variant]"""
import os, signal, sys, time
signal.signal(signal.SIGPIPE, signal.SIG_DFL)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1605_01078_b200 as S
dim = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
v = sys.argv[2] if len(sys.argv) > 2 else "naive2"
g = torch.Generator().manual_seed(0)
A, B, C = ((torch.rand(dim, dim, dtype=torch.float64, generator=g) * 2 - 1).pin_memory().t() for _ in range(3))
ctx = S.Ctx()
ctx.gemm(v[:-1], int(v[-1]), 1.0, A, B, C)
ctx.enable_profiling(True)
t0 = time.perf_counter()
ctx.gemm(v[:-1], int(v[-1]), 1.0, A, B, C)
wall = (time.perf_counter() - t0) * 1e3
prof = ctx.last_profile()
busy = sum(p["ms"] for p in prof)
last_end = max(p["start_ms"] + p["ms"] for p in prof)
print(f"{v} {dim}: wall {wall:.1f} ms, first launch -> last kernel end {last_end:.1f} ms, "
      f"kernel-busy {busy:.1f} ms, launches {len(prof)}")
# coverage: union of kernel intervals (two streams may overlap)
iv = sorted((p["start_ms"], p["start_ms"] + p["ms"]) for p in prof)
cov, cur_s, cur_e = 0.0, None, None
gaps = []
for s_, e_ in iv:
    if cur_e is None or s_ > cur_e:
        if cur_e is not None:
            cov += cur_e - cur_s
            gaps.append((cur_e, s_ - cur_e))
        cur_s, cur_e = s_, e_
    else:
        cur_e = max(cur_e, e_)
cov += cur_e - cur_s
print(f"GPU covered {cov:.1f} ms of {last_end:.1f}; largest idle gaps (at ms, length):",
      [(round(a, 1), round(b, 2)) for a, b in sorted(gaps, key=lambda x: -x[1])[:8]])
print("first 12:", [(p["kernel"][:6], round(p["start_ms"], 2), round(p["ms"], 2)) for p in prof[:12]])
