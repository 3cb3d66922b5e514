"""One strassen_gemm_device call at m = n = k = N (default 65536: A, B, C take 103 GB)
for each given configuration, with an fp64 Freivalds check.  Naive / C at this size
need product groups (their operand sums alone would be 184 GB at level 2).
usage: python tools/huge_call.py [N] [naive2,c2,abc2]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch

import paper_1605_01078_b200 as S
from gpu_util import counter_uniform_torch

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
configs = (sys.argv[2] if len(sys.argv) > 2 else "naive2,c2,abc2").split(",")
A = counter_uniform_torch(1, 0, N, 0, N, 9)
B = counter_uniform_torch(2, 0, N, 0, N, 9)
C = counter_uniform_torch(3, 0, N, 0, N, 9)
g = torch.Generator(device="cuda").manual_seed(9)
x = torch.rand((N, 1), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
abx = A @ (B @ x)
den = (torch.linalg.norm(A) * torch.linalg.norm(B) * torch.linalg.norm(x)).item()
ctx = S.Ctx()
ctx.set_max_level(3)
for cfg in configs:
    v, L = cfg[:-1], int(cfg[-1])
    c0x = C @ x
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.gemm_device(v, L, 1.0, A, B, C)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    frei = (torch.linalg.norm(C @ x - c0x - abx) / den).item()
    print(json.dumps({"m=n=k": N, "config": cfg, "ms": ms,
                      "effective_tflops": 2.0 * N ** 3 / (ms * 1e-3) / 1e12,
                      "launches": ctx.last_launches(), "freivalds_fp64": frei,
                      "workspace_gb": ctx.workspace_bytes() / 1e9}), flush=True)
