#!/bin/bash
# classical stream-K extended to 2-4 waves of tiles: correctness vs cuBLAS, then the mid-size scan
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1605_01078_b200 as S
ctx = S.Ctx()
worst = 0
for (m, n, k) in [(2304,2304,2304),(2432,2432,2432),(2560,2560,300),(2816,2816,2816),(2944,2700,1000),(2301,2417,777),(3000,3000,3000),(2304,4608,512)]:
    g = torch.Generator(device="cuda").manual_seed(m+n+k)
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g)*2-1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g)*2-1).t()
    C0 = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g)*2-1).t()
    ref = C0 - 0.5 * (A @ B)
    outs = []
    for rep in range(2):
        C = C0.t().clone().t()
        ctx.gemm_device("dgemm", 0, -0.5, A, B, C)
        torch.cuda.synchronize()
        outs.append(C)
    e = ((outs[0]-ref).norm()/(A.norm()*B.norm())).item()
    worst = max(worst, e)
    print(m, n, k, "normwise %.2e" % e, "repeatable", torch.equal(outs[0], outs[1]), "launches", ctx.last_launches(), flush=True)
print("worst", worst)
PY
for w in 0 1; do echo "== STREAMK_WIDE=$w"; STRASSEN_B200_STREAMK_WIDE=$w N=20 timeout 900 python tools/small_sizes.py 2176,2304,2432,2560,2688,2816,2944,3072,3328 dgemm0 2>&1 | grep -v cublas | sed 's/(executed.*kernels/kernels/' | sed 's/| single.*//'; done | tee gpurun_out/r02_streamk_wide_ab.log
