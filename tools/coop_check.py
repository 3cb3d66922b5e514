"""Checksums of small-size results (the fixup paths): run once per setting of
STRASSEN_B200_COOP / STRASSEN_B200_LIB and diff the outputs -- the cooperative fixup
sums the pieces in the same order as the single-owner one, so every line must match."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

shapes = [(768, 768, 768), (1000, 1000, 1000), (1024, 1024, 1024), (1280, 1280, 1280),
          (1536, 1536, 1536), (2048, 2048, 2048), (777, 1031, 515), (640, 512, 4096),
          (512, 512, 512), (2560, 1024, 768), (1024, 1024, 8192)]
confs = [("dgemm", 0), ("abc", 1), ("ab", 1), ("naive", 1), ("c", 1), ("abc", 2), ("c", 2)]
ctx = S.Ctx()
for m, n, k in shapes:
    g = torch.Generator(device="cuda").manual_seed(m + 3 * n + 7 * k)
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    ref = C0 + A @ B
    for v, L in confs:
        for layout in ("col", "row"):
            # (m, n) with strides (1, m) / (n, 1); fresh copies of C0
            C = C0.t().clone().t() if layout == "col" else C0.contiguous().clone()
            ctx.gemm_device(v, L, 1.0, A, B, C)
            torch.cuda.synchronize()
            err = ((C - ref).norm() / (A.norm() * B.norm())).item()
            h = hashlib.sha1(C.contiguous().cpu().numpy().tobytes()).hexdigest()[:16]
            print(f"{m}x{n}x{k} {v}{L} {layout} {h} {'ok' if err < 5e-12 else 'BAD %.3e' % err}",
                  flush=True)
