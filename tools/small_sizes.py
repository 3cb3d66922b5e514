"""Small sizes (BASELINE config 1 and the bottom of the square sweep): per-call time of
the library's configurations and of cuBLAS DGEMM (torch.addmm, C := A B + C), each
timed two ways with CUDA events: back to back (N calls, steady state) and as a single
call between synchronisations.  Also the library's per-launch kernel times.

usage: python tools/small_sizes.py [1024,1536,2048] [abc1,dgemm0,...]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,1536,2048").split(",")]
confs = (sys.argv[2] if len(sys.argv) > 2 else
         "dgemm0,abc1,ab1,naive1,c1,abc2,ab2,naive2,c2").split(",")
N = int(os.environ.get("N", "50"))
PEAK = 37.05


def executed(v, L, d):
    if L == 0:
        return 2.0 * d ** 3
    q = d >> L
    mul, aa, ba, cu = {1: (7, 5, 5, 12), 2: (49, 95, 95, 144)}[L]
    f = mul * 2.0 * q ** 3
    if v in ("abc", "ab"):
        f += 2.0 * (aa + ba) * q * q
    if v in ("abc", "c"):
        f += 2.0 * cu * q * q
    return f


def timed(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(N):
        fn()
    e1.record()
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / N * 1e3
    single = []
    for _ in range(15):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        single.append(e0.elapsed_time(e1) * 1e3)
    return b2b, statistics.median(single)


ctx = S.Ctx()
for d in sizes:
    g = torch.Generator(device="cuda").manual_seed(d)
    A, B, C = ((torch.rand(d, d, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
               for _ in range(3))
    flops = 2.0 * d ** 3
    b2b, one = timed(lambda: C.addmm_(A, B))
    print(f"{d} cublas: back-to-back {b2b:7.1f} us {flops / b2b / 1e6:6.2f} TF/s | "
          f"single {one:7.1f} us {flops / one / 1e6:6.2f} TF/s", flush=True)
    for vl in confs:
        v, L = vl[:-1], int(vl[-1])
        b2b, one = timed(lambda: ctx.gemm_device(v, L, 1.0, A, B, C))
        ctx.enable_profiling(True)
        ctx.gemm_device(v, L, 1.0, A, B, C)
        torch.cuda.synchronize()
        prof = ctx.last_profile()
        ctx.enable_profiling(False)
        kern = " ".join(f"{p['kernel'][:6]}={p['ms'] * 1e3:.1f}" for p in prof)
        mm = sum(p["ms"] for p in prof if p["kernel"] == "mm_kernel") * 1e-3
        frac = executed(v, L, d) / b2b / 1e6 / PEAK
        print(f"{d} {vl}: back-to-back {b2b:7.1f} us {flops / b2b / 1e6:6.2f} TF/s "
              f"(executed {frac:.2f} of peak) | single {one:7.1f} us {flops / one / 1e6:6.2f} TF/s"
              f" | kernels(us) {kern} mm {executed(v, L, d) / max(mm, 1e-9) / 1e12 / PEAK:.2f}",
              flush=True)
