"""Epilogue phases of a one-unit-per-CTA fused launch (SB200_TRACE build): per CTA the
time from entry to mainloop end, first stage written, ticket held, reduce-adds issued,
reductions complete, exit.   usage: python tools/cta_trace_epi.py variant level m n k"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["STRASSEN_B200_LIB"] = "libstrassen_b200_trace.so"
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

v, L, m, n, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
C = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
ctx = S.Ctx()
for _ in range(2):
    ctx.gemm_device(v, L, 1.0, A, B, C)
torch.cuda.synchronize()
buf = torch.zeros(8192 * 32, dtype=torch.int64, device="cuda")
os.environ["STRASSEN_B200_TRACE_PTR"] = str(buf.data_ptr())
ctx.enable_profiling(True)
ctx.gemm_device(v, L, 1.0, A, B, C)
torch.cuda.synchronize()
prof = ctx.last_profile()
del os.environ["STRASSEN_B200_TRACE_PTR"]
t = buf.view(8192, 32).cpu().tolist()
rows = [r for r in t if r[0] > 0 and r[31] > 0 and r[2] > 0]
print(f"{v}{L} {m}x{n}x{k}: {len(rows)} traced CTAs; kernels "
      f"{[(p['kernel'], round(p['ms'] * 1e3, 1)) for p in prof]} us")
names = [("mainloop", 1, 2), ("-> first stage written", 2, 20), ("ticket wait", 20, 21),
         ("-> reduce-adds issued", 21, 22), ("completion wait", 22, 23), ("-> exit", 23, 31),
         ("whole CTA", 0, 31), ("epilogue (mainloop end -> exit)", 2, 31)]
for name, a, b in names:
    d = [(r[b] - r[a]) / 1e3 for r in rows if r[a] > 0 and r[b] > 0]
    if d:
        d.sort()
        print(f"  {name:34s} n={len(d):5d} median {statistics.median(d):7.2f} us  mean "
              f"{statistics.mean(d):7.2f}  p90 {d[int(0.9 * len(d))]:7.2f}")
