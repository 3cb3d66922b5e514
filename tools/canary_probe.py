"""Clipped-destination probe: C embedded in a larger host buffer; reports writes outside
the view and the max error inside, per variant (tools/canary_probe.py)."""
import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_1605_01078_b200 as S
from gpu_util import inputs
ctx = S.Ctx()
m, n, k = 133, 77, 150
a, b, _ = inputs(m, n, k, (8, 9, 10))
sentinel = -777.25
for v, L in [("abc", 2), ("c", 2), ("c", 1), ("abc", 1), ("dgemm", 0), ("ab", 2)]:
    buf = np.full((m + 9, n + 7), sentinel, order="F")
    c = buf[3:3 + m, 2:2 + n]
    c[...] = 0.0
    ctx.gemm(v, L, 1.0, a, b, c)
    outside = buf.copy()
    outside[3:3 + m, 2:2 + n] = sentinel
    bad = np.argwhere(outside != sentinel)
    ref = a @ b
    print(v, L, "outside writes:", len(bad), bad[:6].tolist(), "max err inside", float(np.abs(c - ref).max()), "launches", ctx.last_launches(), flush=True)
