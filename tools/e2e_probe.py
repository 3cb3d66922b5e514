"""e2e probe: strassen_gemm through the C ABI with pinned host buffers.

usage: e2e_probe.py [dim] [naive2,abc1,...] [grid,grid,...]
grid = "RxC" window grid (STRASSEN_B200_WINDOWS), "off" = no pipelining, "auto" = planner.
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1605_01078_b200 as S
dim = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["naive2", "abc1", "dgemm0"]
grids = sys.argv[3].split(",") if len(sys.argv) > 3 else ["auto"]
ctx = S.Ctx()
g = torch.Generator().manual_seed(0)
A, B, C = ((torch.rand(dim, dim, dtype=torch.float64, generator=g) * 2 - 1).pin_memory().t() for _ in range(3))
for v in variants:
    for grid in grids:
        os.environ.pop("STRASSEN_B200_WINDOWS", None)
        ctx.set_pipelining(grid != "off")
        if grid not in ("off", "auto"):
            os.environ["STRASSEN_B200_WINDOWS"] = grid
        ctx.gemm(v[:-1], int(v[-1]), 1.0, A, B, C)
        t0 = time.perf_counter()
        for _ in range(3):
            ctx.gemm(v[:-1], int(v[-1]), 1.0, A, B, C)
        dt = (time.perf_counter() - t0) / 3
        print(f"{dim} {v} grid={grid}: e2e {dt*1e3:.1f} ms  {2*dim**3/dt/1e12:.2f} TF/s "
              f"launches={ctx.last_launches()}", flush=True)
