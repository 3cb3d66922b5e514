"""One device-resident call (for ncu captures): run_once.py variant level m [n k]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1605_01078_b200 as S
v, L, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 else m
k = int(sys.argv[5]) if len(sys.argv) > 5 else m
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
C = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
ctx = S.Ctx()
if L == 3:
    ctx.set_max_level(3)
ctx.gemm_device(v, L, 1.0, A, B, C)
torch.cuda.synchronize()
print("ok", ctx.last_launches())
if os.environ.get("PROFILE"):
    ctx.enable_profiling(True)
    for _ in range(3):
        ctx.gemm_device(v, L, 1.0, A, B, C)
    torch.cuda.synchronize()
    prof = ctx.last_profile()
    print(" ".join(f"{p['kernel']}={p['ms']:.3f}" for p in prof))
    tot = {}
    for p in prof:
        tot[p["kernel"]] = tot.get(p["kernel"], 0.0) + p["ms"]
    span = max(p["start_ms"] + p["ms"] for p in prof)
    print("totals:", {k: round(v, 3) for k, v in tot.items()}, "span_ms:", round(span, 3),
          "sum_ms:", round(sum(tot.values()), 3))
