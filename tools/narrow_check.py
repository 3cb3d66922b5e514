"""Checksums of single-term programs at sizes whose quadrants end in half a tile: run with
STRASSEN_B200_NARROW=0 and =1 and diff (narrow and wide tiles accumulate every element
over k in the same order, so the lines should match)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01078_b200 as S  # noqa: E402

ctx = S.Ctx()
for d in (2816, 3840, 4864, 6400):
    g = torch.Generator(device="cuda").manual_seed(d)
    A = (torch.rand(d, d, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(d, d, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(d, d, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    for v, L in (("c", 2), ("naive", 2), ("c", 1), ("naive", 1), ("ab", 2), ("ab", 1), ("abc", 2),
                 ("dgemm", 0)):
        C = C0.t().clone().t()
        ctx.gemm_device(v, L, 1.0, A, B, C)
        torch.cuda.synchronize()
        print(d, v, L, hashlib.sha1(C.contiguous().cpu().numpy().tobytes()).hexdigest()[:16], flush=True)
