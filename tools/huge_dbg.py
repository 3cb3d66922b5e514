"""Grouped-product calls at a large size under several memory caps (debug)."""
import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
import paper_1605_01078_b200 as S
from gpu_util import counter_uniform_torch
N = int(sys.argv[1])
A = counter_uniform_torch(1, 0, N, 0, N, 9); B = counter_uniform_torch(2, 0, N, 0, N, 9); C = counter_uniform_torch(3, 0, N, 0, N, 9)
torch.cuda.synchronize()
print("mem_get_info GB", [x / 1e9 for x in torch.cuda.mem_get_info()], "torch reserved GB", torch.cuda.memory_reserved() / 1e9, flush=True)
ctx = S.Ctx()
for cap in [None, str(60 << 30), str(30 << 30)]:
    if cap: os.environ["STRASSEN_B200_MEM_CAP"] = cap
    try:
        ctx.gemm_device("naive", 2, 1.0, A, B, C); torch.cuda.synchronize()
        print("cap", cap, "ok launches", ctx.last_launches(), "ws GB", ctx.workspace_bytes() / 1e9, flush=True)
    except Exception as e:
        print("cap", cap, "failed", e, S.lib().strassen_last_error().decode() if hasattr(S.lib(), "strassen_last_error") else "", "ws GB", ctx.workspace_bytes() / 1e9, [x / 1e9 for x in torch.cuda.mem_get_info()], flush=True)
