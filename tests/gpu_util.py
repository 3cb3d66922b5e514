"""Shared helpers for the -m gpu parity tests (checker side: the oracle)."""
import numpy as np

import oracle_lib as O

# the reference's seven configurations plus the B200 "C" variant at both levels
CONFIGS = [("dgemm", 0), ("abc", 1), ("ab", 1), ("naive", 1), ("abc", 2), ("ab", 2), ("naive", 2),
           ("c", 1), ("c", 2)]
# BASELINE.json north star: normwise ||C - C_ref||_F / (||A||_F ||B||_F)
NORMWISE_TOL = {0: 1e-12, 1: 1e-12, 2: 5e-12}
# the reference's own tolerance on rel_frobenius_error (test_capi.cpp:92, test_strassen.cpp:79)
REL_TOL = 1e-11


def inputs(m, n, k, seeds=(1, 2, 3), layout="col"):
    a = O.fill_uniform(m * k, seeds[0])
    b = O.fill_uniform(k * n, seeds[1])
    c = O.fill_uniform(m * n, seeds[2])
    if layout == "row":
        return a.reshape(m, k), b.reshape(k, n), c.reshape(m, n)
    return (np.asfortranarray(a.reshape(k, m).T), np.asfortranarray(b.reshape(n, k).T),
            np.asfortranarray(c.reshape(n, m).T))


def oracle_result(variant, level, alpha, a, b, c0, use_reference_gemm=None):
    """Reference arithmetic on the same inputs: the triple-loop oracle for small
    problems, the reference blocked DGEMM restatement above (bench_lib.cpp:208-221)."""
    c = np.array(c0, copy=True, order="F")
    m, k = a.shape
    n = b.shape[1]
    if use_reference_gemm is None:
        use_reference_gemm = max(m, n, k) <= 400
    if use_reference_gemm:
        O.reference_gemm(alpha, a, b, c)
    else:
        O.strassen_gemm("dgemm", 0, alpha, a, b, c)
    return c


def errors(c_gpu, c_ref, c0, a, b):
    """(normwise, rel_frobenius) of the GPU result against the oracle."""
    nw = O.normwise_error(np.asarray(c_gpu), np.asarray(c_ref), a, b)
    rel = O.rel_frobenius_error(np.ascontiguousarray(c_gpu), np.ascontiguousarray(c_ref))
    return nw, rel


def check(variant, level, c_gpu, c_ref, c0, a, b):
    nw, rel = errors(c_gpu, c_ref, c0, a, b)
    assert nw <= NORMWISE_TOL[level], (variant, level, nw)
    assert rel <= REL_TOL, (variant, level, rel)
    return nw, rel


def freivalds(alpha, a, b, c0, c, seed=0):
    """Size-independent check: ||C x - C0 x - alpha A (B x)|| / (||A||_F ||B||_F ||x||)
    in long double, O(n^2)."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, size=(b.shape[1], 2)).astype(np.longdouble)
    lhs = np.asarray(c, dtype=np.longdouble) @ x - np.asarray(c0, dtype=np.longdouble) @ x
    rhs = alpha * (np.asarray(a, dtype=np.longdouble) @ (np.asarray(b, dtype=np.longdouble) @ x))
    num = np.linalg.norm((lhs - rhs).astype(np.float64))
    den = np.linalg.norm(a) * np.linalg.norm(b) * np.linalg.norm(x.astype(np.float64))
    return float(num / den)


# ---- counter-based RNG (distributed sizes regenerate any tile) --------
# value(id, i, j) = 2 * h / 2^32 - 1 with h a 32-bit mix of (seed, matrix id, global row,
# global column); the same integer arithmetic in numpy (oracle side) and torch (GPU
# side), so shards and oracle tiles of a 65536^3 problem never need the full matrices.
M32 = 0xFFFFFFFF


def _mix32(x, xp_and):
    x = xp_and(x ^ (x >> 16), M32)
    x = xp_and(x * 0x7FEB352D, M32)
    x = xp_and(x ^ (x >> 15), M32)
    x = xp_and(x * 0x846CA68B, M32)
    return xp_and(x ^ (x >> 16), M32)


def counter_uniform_np(mid, r0, rows, c0, cols, seed=0):
    """Column-major (Fortran) rows x cols tile of matrix `mid` at (r0, c0), uniform[-1,1)."""
    import numpy as np
    i = np.arange(r0, r0 + rows, dtype=np.int64)[:, None]
    j = np.arange(c0, c0 + cols, dtype=np.int64)[None, :]
    with np.errstate(over="ignore"):
        x = (i * 0x9E3779B1 + j * 0x85EBCA77 + mid * 0xC2B2AE3D + seed) & M32
        h = _mix32(x, np.bitwise_and)
    return np.asfortranarray(h.astype(np.float64) * (2.0 / 4294967296.0) - 1.0)


def counter_uniform_torch(mid, r0, rows, c0, cols, seed=0, device="cuda", out=None):
    """Same values as counter_uniform_np, generated on the GPU in column chunks into a
    column-major (rows x cols) view `out` (allocated if None)."""
    import torch
    if out is None:
        out = torch.empty((cols, rows), dtype=torch.float64, device=device).t()
    i = torch.arange(r0, r0 + rows, dtype=torch.int64, device=device)[:, None]
    step = max(1, (1 << 27) // max(rows, 1))
    for cs in range(0, cols, step):
        ce = min(cols, cs + step)
        j = torch.arange(c0 + cs, c0 + ce, dtype=torch.int64, device=device)[None, :]
        x = (i * 0x9E3779B1 + j * 0x85EBCA77 + mid * 0xC2B2AE3D + seed) & M32
        h = _mix32(x, torch.bitwise_and)
        out[:, cs:ce] = h.to(torch.float64) * (2.0 / 4294967296.0) - 1.0
    return out
