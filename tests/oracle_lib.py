"""ctypes bindings to the parity checker (test infrastructure only).

Loads oracle/_build/libstrassen_oracle.so (the C restatement, see
oracle/strassen_oracle.c) and, when present, oracle/_ref/libstrassen_ref.so
(the reference library itself, compiled from /root/reference/proj/src by
oracle/Makefile).  Only tests/, __graft_entry__.smoke() and bench.py's
reference / cpu_baseline legs use this module.
"""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libstrassen_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libstrassen_ref.so")

_dp = C.POINTER(C.c_double)
_L = C.c_long


def _ptr(x):
    return x.ctypes.data_as(_dp)


def build():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=True)


class SoEntry(C.Structure):
    _fields_ = [("na", C.c_int), ("nb", C.c_int), ("nc", C.c_int)] + [
        (f, C.c_int * 8) for f in ("aq", "as_", "bq", "bs", "cq", "cs")
    ]


_oracle = None


def oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        lib.so_fill_uniform.argtypes = [_dp, _L, C.c_uint64, C.c_double, C.c_double]
        lib.so_mt19937_64.argtypes = [C.c_uint64, _L, C.POINTER(C.c_uint64)]
        lib.so_reference_gemm.argtypes = [_L, _L, _L, C.c_double, _dp, _L, _L, _dp, _L, _L, _dp, _L, _L]
        lib.so_rel_frobenius_error.argtypes = [_L, _L, _dp, _L, _L, _dp, _L, _L]
        lib.so_rel_frobenius_error.restype = C.c_double
        lib.so_normwise_error.argtypes = [_L, _L, _L, _dp, _dp, _dp, _dp]
        lib.so_normwise_error.restype = C.c_double
        lib.so_table.argtypes = [C.c_int, C.POINTER(SoEntry)]
        lib.so_strassen_gemm.argtypes = [C.c_int, C.c_int, _L, _L, _L, C.c_double,
                                         _dp, _L, _L, _dp, _L, _L, _dp, _L, _L, _L]
        _oracle = lib
    return _oracle


def fill_uniform(n, seed, lo=-1.0, hi=1.0):
    """std::mt19937_64(seed) + uniform_real_distribution<double>(lo, hi)."""
    out = np.empty(int(n), dtype=np.float64)
    oracle().so_fill_uniform(_ptr(out), int(n), seed, lo, hi)
    return out


def mt19937_64(seed, n):
    out = np.empty(int(n), dtype=np.uint64)
    oracle().so_mt19937_64(seed, int(n), out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def table(level):
    """List of (a_terms, b_terms, c_terms) with (quadrant, coeff) pairs."""
    buf = (SoEntry * 343)()
    n = oracle().so_table(level, buf)
    assert n > 0
    out = []
    for e in buf[:n]:
        out.append((
            [(e.aq[u], e.as_[u]) for u in range(e.na)],
            [(e.bq[u], e.bs[u]) for u in range(e.nb)],
            [(e.cq[u], e.cs[u]) for u in range(e.nc)],
        ))
    return out


def _strides(x):
    return x.strides[0] // 8, x.strides[1] // 8


def reference_gemm(alpha, a, b, c):
    """c += alpha a b (in place), matrix.cpp:37-52 semantics."""
    m, k = a.shape
    n = b.shape[1]
    rc = oracle().so_reference_gemm(m, n, k, alpha, _ptr(a), *_strides(a), _ptr(b), *_strides(b),
                                    _ptr(c), *_strides(c))
    assert rc == 0
    return c


VARIANTS = {"dgemm": 0, "abc": 1, "ab": 2, "naive": 3}


def strassen_gemm(variant, level, alpha, a, b, c, kc=256):
    """c += alpha a b through the restated reference algorithm (in place)."""
    m, k = a.shape
    n = b.shape[1]
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    rc = oracle().so_strassen_gemm(v, level, m, n, k, alpha, _ptr(a), *_strides(a), _ptr(b),
                                   *_strides(b), _ptr(c), *_strides(c), kc)
    assert rc == 0, rc
    return c


def rel_frobenius_error(t, r):
    return oracle().so_rel_frobenius_error(t.shape[0], t.shape[1], _ptr(t), *_strides(t), _ptr(r),
                                           *_strides(r))


def normwise_error(c_test, c_ref, a, b):
    """||C_test - C_ref||_F / (||A||_F ||B||_F) (BASELINE.json tolerance metric)."""
    ct = np.ascontiguousarray(c_test, dtype=np.float64)
    cr = np.ascontiguousarray(c_ref, dtype=np.float64)
    aa = np.ascontiguousarray(a, dtype=np.float64)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    return oracle().so_normwise_error(ct.shape[0], ct.shape[1], aa.shape[1], _ptr(ct), _ptr(cr),
                                      _ptr(aa), _ptr(bb))


# ----------------------------------------------------------- reference .so
class RefStrassen:
    """The reference library itself (oracle/_ref/libstrassen_ref.so)."""

    def __init__(self, path=REF_SO):
        lib = C.CDLL(path)
        lib.strassen_ctx_create.argtypes = [C.POINTER(C.c_void_p)]
        lib.strassen_ctx_destroy.argtypes = [C.c_void_p]
        lib.strassen_ctx_set_threads.argtypes = [C.c_void_p, C.c_int]
        lib.strassen_ctx_enable_counters.argtypes = [C.c_void_p, C.c_int]
        lib.strassen_ctx_get_counters.argtypes = [C.c_void_p, C.POINTER(C.c_int64 * 19)]
        lib.strassen_gemm.argtypes = [C.c_void_p, C.c_int, C.c_int, _L, _L, _L, C.c_double,
                                      _dp, _L, _L, _dp, _L, _L, _dp, _L, _L]
        lib.strassen_reference_gemm.argtypes = [_L, _L, _L, C.c_double, _dp, _L, _L, _dp, _L, _L,
                                                _dp, _L, _L]
        self.lib = lib
        self.ctx = C.c_void_p()
        assert lib.strassen_ctx_create(C.byref(self.ctx)) == 0

    @staticmethod
    def available(path=REF_SO):
        return os.path.exists(path)

    def set_threads(self, t):
        assert self.lib.strassen_ctx_set_threads(self.ctx, int(t)) == 0

    def enable_counters(self, on=True):
        assert self.lib.strassen_ctx_enable_counters(self.ctx, int(on)) == 0

    def counters(self):
        out = (C.c_int64 * 19)()
        assert self.lib.strassen_ctx_get_counters(self.ctx, C.byref(out)) == 0
        return list(out)

    def gemm(self, variant, level, alpha, a, b, c):
        m, k = a.shape
        n = b.shape[1]
        v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
        rc = self.lib.strassen_gemm(self.ctx, v, level, m, n, k, alpha, _ptr(a), *_strides(a),
                                    _ptr(b), *_strides(b), _ptr(c), *_strides(c))
        assert rc == 0, rc
        return c

    def gemm_raw(self, variant, level, m, n, k, alpha, a, rsa, csa, b, rsb, csb, c, rsc, csc):
        return self.lib.strassen_gemm(self.ctx, variant, level, m, n, k, alpha, a, rsa, csa, b,
                                      rsb, csb, c, rsc, csc)

    def __del__(self):
        try:
            self.lib.strassen_ctx_destroy(self.ctx)
        except Exception:
            pass
