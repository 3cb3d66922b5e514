"""Debug/probe: time and check gemm_device across sizes (Freivalds vs torch fp64)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1605_01078_b200 as S

ctx = S.Ctx()
variants = [v for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["dgemm0", "abc1", "abc2"])]
for dim in [int(x) for x in sys.argv[1].split(",")]:
    g = torch.Generator(device="cuda").manual_seed(dim)
    A = (torch.rand(dim, dim, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(dim, dim, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(dim, dim, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    x = torch.rand(dim, 1, dtype=torch.float64, device="cuda", generator=g)
    want = C0 @ x + A @ (B @ x)
    for vl in variants:
        v, L = vl[:-1], int(vl[-1])
        C = C0.clone().t().contiguous().t()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.gemm_device(v, L, 1.0, A, B, C)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        err = (torch.linalg.norm(C @ x - want) / (torch.linalg.norm(A) * torch.linalg.norm(B) * torch.linalg.norm(x))).item()
        print(f"{dim} {vl}: {ms:.3f} ms  {2*dim**3/ms/1e9:.2f} TF/s  freivalds {err:.2e}  launches {ctx.last_launches()}", flush=True)
