"""A/B of the stream pass forms (shared-memory vs register accumulators): stream-kernel
time per call and bitwise equality of the results."""
import os, sys, subprocess
sys.path.insert(0, '.')
import torch
import paper_1605_01078_b200 as S
res = {}
for v, L, d in [("naive", 2, 16384), ("naive", 1, 8192), ("ab", 2, 8192), ("naive", 2, 4097), ("naive", 3, 16384)]:
    outs = []
    for fixed in ("0", "1"):
        code = f'''
import sys; sys.path.insert(0, ".")
import torch, paper_1605_01078_b200 as S
g = torch.Generator(device="cuda").manual_seed(7)
A, B, C = ((torch.rand({d}, {d}, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t() for _ in range(3))
ctx = S.Ctx(); ctx.set_max_level(3)
ctx.gemm_device("{v}", {L}, 1.0, A, B, C); torch.cuda.synchronize()
ctx.enable_profiling(True)
C2 = C.clone().t().contiguous().t()
ctx.gemm_device("{v}", {L}, 1.0, A, B, C2); torch.cuda.synchronize()
st = sum(p["ms"] for p in ctx.last_profile() if p["kernel"] == "stream_gather_kernel")
torch.save(C2.cpu(), "/tmp/c_{fixed}.pt")
print(st)
'''
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, STRASSEN_B200_STREAM_FIXED=fixed), capture_output=True, text=True)
        outs.append(float(out.stdout.strip().split()[-1]) if out.returncode == 0 else out.stderr[-300:])
    eq = torch.equal(torch.load("/tmp/c_0.pt"), torch.load("/tmp/c_1.pt"))
    print(v, L, d, "stream ms smem/fixed:", outs, "bitwise equal:", eq, flush=True)
