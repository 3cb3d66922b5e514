"""Per-CTA timeline of one mm_kernel launch (the SB200_TRACE build,
`make -C paper_1605_01078_b200/csrc trace`): %globaltimer stamps at CTA entry, each
unit's start and epilogue start, and CTA exit.

usage: python tools/cta_trace.py variant level m [n k]     (prints the breakdown)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["STRASSEN_B200_LIB"] = "libstrassen_b200_trace.so"
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

v, L, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 else m
k = int(sys.argv[5]) if len(sys.argv) > 5 else m
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
C = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
ctx = S.Ctx()
for _ in range(5):
    ctx.gemm_device(v, L, 1.0, A, B, C)
torch.cuda.synchronize()
buf = torch.zeros(8192 * 32, dtype=torch.int64, device="cuda")
os.environ["STRASSEN_B200_TRACE_PTR"] = str(buf.data_ptr())
ctx.enable_profiling(True)
ctx.gemm_device(v, L, 1.0, A, B, C)
torch.cuda.synchronize()
prof = ctx.last_profile()
del os.environ["STRASSEN_B200_TRACE_PTR"]
t = buf.view(8192, 32).cpu()
ctas = [r for r in t.tolist() if r[0] > 0]
t0 = min(r[0] for r in ctas)
us = lambda x: (x - t0) / 1e3  # noqa: E731
entry = [us(r[0]) for r in ctas]
exit_ = [us(r[31]) for r in ctas]
main, epi, units = [], [], []
for r in ctas:
    ev = [x for x in r[1:31]]
    nu = 0
    mt = et = 0.0
    for i in range(15):
        s, e = ev[2 * i], ev[2 * i + 1]
        if s == 0:
            break
        nxt = ev[2 * i + 2] if 2 * i + 2 < 30 and ev[2 * i + 2] > 0 else r[31]
        if e > 0:
            mt += (e - s) / 1e3
            et += (nxt - e) / 1e3
        nu += 1
    main.append(mt)
    epi.append(et)
    units.append(nu)
print(f"{v}{L} {m}x{n}x{k}: {len(ctas)} CTAs; kernels {[(p['kernel'], round(p['ms'] * 1e3, 1)) for p in prof]} us")
print(f"  CTA entry spread {max(entry) - min(entry):.1f} us (median {statistics.median(entry):.1f});"
      f" exit: min {min(exit_):.1f} median {statistics.median(exit_):.1f} max {max(exit_):.1f} us")
print(f"  per CTA: units mean {statistics.mean(units):.2f} max {max(units)};"
      f" mainloop mean {statistics.mean(main):.1f} max {max(main):.1f} us;"
      f" epilogue+fixup mean {statistics.mean(epi):.1f} max {max(epi):.1f} us;"
      f" active mean {statistics.mean(x - y for x, y in zip(exit_, entry)):.1f} us")
slow = sorted(range(len(ctas)), key=lambda i: -exit_[i])[:5]
for i in slow:
    r = ctas[i]
    evs = [round(us(x), 1) for x in r[:31] if x > 0] + [round(us(r[31]), 1)]
    print(f"  late CTA {i}: units {units[i]} main {main[i]:.1f} epi {epi[i]:.1f}: {evs}")
