"""Probe: time gemm_device across sizes/variants (median of reps) with a
Freivalds check, and record SM clocks during the run."""
import os
import statistics
import subprocess
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1605_01078_b200 as S

reps = int(os.environ.get("REPS", "3"))
ctx = S.Ctx()
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["dgemm0", "abc1", "abc2"]
clk = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                        stderr=subprocess.DEVNULL, text=True)
threading.Thread(target=lambda: [clk.append(l.strip()) for l in proc.stdout], daemon=True).start()
for spec in sys.argv[1].split(","):
    m, n, k = (int(v) for v in spec.split("x")) if "x" in spec else (int(spec),) * 3
    dim = spec
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    x = torch.rand(n, 1, dtype=torch.float64, device="cuda", generator=g)
    want = C0 @ x + A @ (B @ x)
    for vl in variants:
        v, L = vl[:-1], int(vl[-1])
        times = []
        for r in range(reps + 1):
            C = C0.clone().t().contiguous().t()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.gemm_device(v, L, 1.0, A, B, C)
            e1.record()
            torch.cuda.synchronize()
            if r > 0 or reps == 0:
                times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        err = (torch.linalg.norm(C @ x - want) /
               (torch.linalg.norm(A) * torch.linalg.norm(B) * torch.linalg.norm(x))).item()
        print(f"{dim} {vl}: {ms:.3f} ms  {2*m*n*k/ms/1e9:.2f} TF/s  (min {min(times):.3f})  "
              f"freivalds {err:.2e}  launches {ctx.last_launches()}", flush=True)
proc.terminate()
sm = [float(l.split(",")[0]) for l in clk if l and l.split(",")[0].strip().replace(".", "").isdigit()]
pw = [float(l.split(",")[1]) for l in clk if l and len(l.split(",")) > 1 and l.split(",")[1].strip().replace(".", "").isdigit()]
if sm:
    print(f"clocks: sm median {statistics.median(sm):.0f} MHz min {min(sm):.0f} max {max(sm):.0f}; "
          f"power max {max(pw) if pw else 0:.0f} W; reasons {sorted(set(l.split(',')[-1].strip() for l in clk if l))}")
