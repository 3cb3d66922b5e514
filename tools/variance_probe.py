"""Run-to-run spread of single device calls (10 repetitions each) at one size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1605_01078_b200 as S

d = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cfgs = (sys.argv[2] if len(sys.argv) > 2 else "c1,c2,naive2,dgemm0,abc2").split(",")
g = torch.Generator(device="cuda").manual_seed(d)
A, B, C = ((torch.rand(d, d, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
           for _ in range(3))
ctx = S.Ctx()
ctx.set_max_level(3)
for cfg in cfgs:
    v, L = cfg[:-1], int(cfg[-1])
    ts = []
    for r in range(11):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.gemm_device(v, L, 1.0, A, B, C)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    print(cfg, " ".join(f"{t:.1f}" for t in ts), flush=True)
