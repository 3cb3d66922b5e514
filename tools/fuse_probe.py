"""Time fused-sum programs with operand sides of > F terms materialised by the sum pass
(STRASSEN_B200_FUSE_MAX = F; 4 = fully fused ABC / AB), and check the result is
bitwise the same for every F.   fuse_probe.py [variant level m n k] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

cases = [("abc", 2, 16384, 16384, 16384), ("ab", 2, 16384, 16384, 16384),
         ("abc", 1, 16384, 16384, 16384), ("abc", 2, 32768, 32768, 1024),
         ("abc", 2, 16384, 16384, 256), ("abc", 2, 16384, 16384, 1024)]
if len(sys.argv) > 1:
    a = sys.argv[1:]
    cases = [(a[i], int(a[i + 1]), int(a[i + 2]), int(a[i + 3]), int(a[i + 4]))
             for i in range(0, len(a), 5)]
fmax = [int(x) for x in os.environ.get("FMAX", "4,2,1").split(",")]
reps = int(os.environ.get("REPS", "3"))
for v, L, m, n, k in cases:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    first = None
    for f in fmax:
        os.environ["STRASSEN_B200_FUSE_MAX"] = str(f)
        ctx = S.Ctx()
        C = C0.clone().t().contiguous().t()
        ctx.gemm_device(v, L, 1.0, A, B, C)  # warm-up, sizes the workspace
        torch.cuda.synchronize()
        if first is None:
            first = C.clone()
        same = torch.equal(C, first)
        ctx.enable_profiling(True)
        best, prof_best = 1e30, None
        for _ in range(reps):
            C.copy_(C0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.gemm_device(v, L, 1.0, A, B, C)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            if t < best:
                best, prof_best = t, ctx.last_profile()
        tf = 2.0 * m * n * k / (best * 1e-3) / 1e12
        parts = " ".join(f"{p['kernel'][:6]}={p['ms']:.3f}" for p in prof_best)
        print(f"{v}{L} {m}x{n}x{k} fuse_max={f}: {best:.3f} ms {tf:.2f} TF/s bitwise_same={same} "
              f"[{parts}]", flush=True)
        ctx.close()
        del C
    del A, B, C0, first
    torch.cuda.empty_cache()
