#!/bin/bash
# classical hybrid (tile-owner waves + stream-K tail): correctness vs cuBLAS, then the scan
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1605_01078_b200 as S
ctx = S.Ctx()
worst = 0
for (m, n, k) in [(3328,3328,3328),(3840,3840,3840),(3584,3584,700),(5632,5632,1024),(3333,3841,515),(4352,3840,2048),(3840,7000,256),(7168,3328,512)]:
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
for w in 0 1; do echo "== STREAMK_WIDE=$w"; STRASSEN_B200_STREAMK_WIDE=$w N=10 timeout 900 python tools/small_sizes.py 3072,3328,3584,3840,4096,4352,4608,4864,5120,5632,6144,6656,7168,7680,8192 dgemm0 2>&1 | grep -v cublas | sed 's/(executed.*kernels/kernels/' | sed 's/| single.*//'; done | tee gpurun_out/r02_tail_ab.log
