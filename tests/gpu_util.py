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
