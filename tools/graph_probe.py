"""strassen_gemm_device under CUDA stream capture: capture one call (after a warm-up
that sizes the workspace) into a CUDA graph, replay it, compare with the eager result
bit for bit, and time graph replays against eager back-to-back calls.

usage: python tools/graph_probe.py [512,768,1024] [dgemm0,abc1,c1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "512,768,1024").split(",")]
confs = (sys.argv[2] if len(sys.argv) > 2 else "dgemm0,abc1,c1").split(",")
N = 50
ctx = S.Ctx()
for d in sizes:
    g = torch.Generator(device="cuda").manual_seed(d)
    A, B, C0 = ((torch.rand(d, d, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
                for _ in range(3))
    for vl in confs:
        v, L = vl[:-1], int(vl[-1])
        C = C0.t().clone().t()
        for _ in range(3):
            ctx.gemm_device(v, L, 1.0, A, B, C)
        torch.cuda.synchronize()
        # eager reference result of ONE call from C0
        Ce = C0.t().clone().t()
        ctx.gemm_device(v, L, 1.0, A, B, Ce)
        torch.cuda.synchronize()
        Cg = C0.t().clone().t()
        graph = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(graph):
                ctx.gemm_device(v, L, 1.0, A, B, Cg, torch.cuda.current_stream())
        except Exception as ex:  # noqa: BLE001
            print(f"{d} {vl}: capture FAILED: {type(ex).__name__}: {str(ex)[:200]}", flush=True)
            torch.cuda.synchronize()
            continue
        Cg.copy_(C0)
        graph.replay()
        torch.cuda.synchronize()
        same = torch.equal(Cg, Ce)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(N):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        tg = e0.elapsed_time(e1) / N * 1e3
        e0.record()
        for _ in range(N):
            ctx.gemm_device(v, L, 1.0, A, B, C)
        e1.record()
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1) / N * 1e3
        print(f"{d} {vl}: graph replay {tg:7.1f} us  eager {te:7.1f} us  bitwise_same={same}",
              flush=True)
