"""paper_1605_01078_b200 -- B200 (sm_100a) Strassen DGEMM behind the reference C ABI.

Python mirror of the reference library's public interface
(/root/reference/proj/include/strassen.h): the same entry points, argument
meaning, status codes and errors, bound with ctypes to the in-tree C-ABI
library ``libstrassen_b200.so`` (built from ``csrc/`` by :func:`build`).
There is no CPU fallback: if the library or a CUDA device is missing, the
compute calls raise.

Operands may be numpy arrays (host memory) or torch tensors (host or CUDA).
Every multiply computes ``C := alpha * A @ B + C`` in place, with the
operands' own strides (a transpose is a stride swap, reference strassen.h:1-6).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

__all__ = [
    "DGEMM", "ABC", "AB", "NAIVE", "StrassenError", "Ctx", "build", "lib", "gemm", "gemm_device",
    "dgemm", "reference_gemm", "rel_error", "table_counts", "effective_gflops", "model_predict",
    "blocking_defaults", "model_params_ivy_bridge", "predicted_counters", "COUNTER_FIELDS",
    "select",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# STRASSEN_B200_LIB: alternative in-tree build (A/B experiments, tools/ab.sh)
LIB_PATH = os.path.join(HERE, os.environ.get("STRASSEN_B200_LIB", "libstrassen_b200.so"))

DGEMM, ABC, AB, NAIVE, C_VARIANT = 0, 1, 2, 3, 4
VARIANT_NAMES = {"dgemm": DGEMM, "abc": ABC, "ab": AB, "naive": NAIVE, "c": C_VARIANT}

OK, ERR_DIMENSION, ERR_PARAM, ERR_DOMAIN, ERR_ALLOC, ERR_NULL, ERR_DEVICE = range(7)

COUNTER_FIELDS = (
    "pack_a_calls", "pack_b_calls", "pack_a_elems", "pack_b_elems", "pack_a_add_flops",
    "pack_b_add_flops", "kernel_calls", "kernel_fma_flops", "kernel_c_elems",
    "kernel_update_flops", "a_plus_passes", "a_plus_elems", "a_plus_flops", "b_plus_passes",
    "b_plus_elems", "b_plus_flops", "c_plus_passes", "c_plus_elems", "c_plus_flops",
)


class Blocking(C.Structure):
    _fields_ = [("mc", C.c_long), ("nc", C.c_long), ("kc", C.c_long), ("mr", C.c_long),
                ("nr", C.c_long)]


class ModelParams(C.Structure):
    _fields_ = [("tau_a", C.c_double), ("tau_b", C.c_double), ("lambda_", C.c_double),
                ("channel_factor", C.c_double)]


class Breakdown(C.Structure):
    _fields_ = [(f, C.c_double) for f in (
        "ta_mul", "ta_a_add", "ta_b_add", "ta_c_add", "tm_a_mul", "tm_b_mul", "tm_c_mul",
        "tm_a_add", "tm_b_add", "tm_c_add", "total")]


class Counters(C.Structure):
    _fields_ = [(f, C.c_int64) for f in COUNTER_FIELDS]


class DistPiece(C.Structure):  # strassen_dist_piece (include/strassen_dist.h)
    _fields_ = [("owner", C.c_int), ("local_off", C.c_long), ("width", C.c_long),
                ("panel_off", C.c_long)]


class StrassenError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = status
        msg = _lib_or_none().strassen_status_str(status).decode() if _lib_or_none() else str(status)
        detail = ""
        if _lib_or_none():
            detail = _lib_or_none().strassen_last_error().decode()
        super().__init__(f"{what}: {msg} ({status}){' - ' + detail if detail else ''}")


def build(verbose=False):
    """Compile libstrassen_b200.so in-tree for sm_100a (nvcc; no GPU needed)."""
    out = subprocess.run(["make", "-C", os.path.join(HERE, "csrc"), "-j4"],
                         capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError("libstrassen_b200 build failed:\n" + (out.stdout or "") + (out.stderr or ""))
    return LIB_PATH


_LIB = None
_dp = C.POINTER(C.c_double)
_L = C.c_long
_ST = C.c_int


def _declare(lib):
    vp = C.c_void_p
    sig = {
        "strassen_ctx_create": (_ST, [C.POINTER(vp)]),
        "strassen_ctx_destroy": (None, [vp]),
        "strassen_ctx_set_blocking": (_ST, [vp, C.POINTER(Blocking)]),
        "strassen_ctx_get_blocking": (_ST, [vp, C.POINTER(Blocking)]),
        "strassen_ctx_set_threads": (_ST, [vp, C.c_int]),
        "strassen_ctx_enable_counters": (_ST, [vp, C.c_int]),
        "strassen_ctx_reset_counters": (_ST, [vp]),
        "strassen_ctx_get_counters": (_ST, [vp, C.POINTER(Counters)]),
        "strassen_gemm": (_ST, [vp, C.c_int, C.c_int, _L, _L, _L, C.c_double, vp, _L, _L, vp, _L,
                                _L, vp, _L, _L]),
        "strassen_reference_gemm": (_ST, [_L, _L, _L, C.c_double, vp, _L, _L, vp, _L, _L, vp, _L,
                                          _L]),
        "strassen_rel_error": (_ST, [_L, _L, vp, _L, _L, vp, _L, _L, _dp]),
        "strassen_model_predict": (_ST, [C.c_int, C.c_int, _L, _L, _L, C.POINTER(Blocking),
                                         C.POINTER(ModelParams), C.POINTER(Breakdown), _dp]),
        "strassen_effective_gflops": (_ST, [_L, _L, _L, C.c_double, _dp]),
        "strassen_model_params_ivy_bridge": (None, [C.POINTER(ModelParams)]),
        "strassen_blocking_defaults": (None, [C.POINTER(Blocking)]),
        "strassen_table_counts": (_ST, [C.c_int, C.POINTER(_L)]),
        "strassen_status_str": (C.c_char_p, [C.c_int]),
        "strassen_gemm_device": (_ST, [vp, vp, C.c_int, C.c_int, _L, _L, _L, C.c_double, vp, _L,
                                       _L, vp, _L, _L, vp, _L, _L]),
        "strassen_dgemm": (_ST, [vp, C.c_int, C.c_int, C.c_char, C.c_char, _L, _L, _L,
                                 C.c_double, vp, _L, vp, _L, C.c_double, vp, _L]),
        "strassen_ctx_set_stream": (_ST, [vp, vp]),
        "strassen_ctx_last_launches": (_ST, [vp, C.POINTER(_L)]),
        "strassen_ctx_workspace_bytes": (_ST, [vp, C.POINTER(_L)]),
        "strassen_count_call": (_ST, [C.c_int, C.c_int, _L, _L, _L, C.POINTER(Blocking),
                                      C.POINTER(Counters)]),
        "strassen_ctx_enable_profiling": (_ST, [vp, C.c_int]),
        "strassen_ctx_set_peeling": (_ST, [vp, C.c_int]),
        "strassen_ctx_set_pipelining": (_ST, [vp, C.c_int]),
        "strassen_ctx_set_max_level": (_ST, [vp, C.c_int]),
        "strassen_ctx_set_fused_terms": (_ST, [vp, C.c_int]),
        "strassen_ctx_set_operand_events": (_ST, [vp, vp, vp, vp]),
        "strassen_ctx_last_profile": (_ST, [vp, C.c_char_p, _L]),
        "strassen_select": (_ST, [_L, _L, _L, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp]),
        "strassen_ctx_select": (_ST, [vp, _L, _L, _L, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      _dp]),
        "strassen_predict_b200": (_ST, [C.c_int, C.c_int, _L, _L, _L, _dp]),
        "strassen_build_info": (C.c_char_p, []),
        "strassen_last_error": (C.c_char_p, []),
        # include/strassen_dist.h
        "strassen_dist_grid": (_ST, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "strassen_dist_default_panel": (_L, [_L]),
        "strassen_dist_panel_pieces": (_ST, [_L, C.c_int, C.c_int, _L, _L, C.c_int,
                                             C.POINTER(DistPiece), _L, C.POINTER(_L)]),
        "strassen_dist_unique_id": (_ST, [vp]),
        "strassen_dist_create": (_ST, [C.POINTER(vp), vp, vp, C.c_int, C.c_int, C.c_int, C.c_int]),
        "strassen_dist_create_from_comm": (_ST, [C.POINTER(vp), vp, vp, C.c_int, C.c_int]),
        "strassen_dist_create_custom": (_ST, [C.POINTER(vp), vp, vp, C.c_int, C.c_int, C.c_int]),
        "strassen_dist_mailbox_create": (_ST, [C.POINTER(vp)]),
        "strassen_dist_mailbox_destroy": (None, [vp]),
        "strassen_dist_mailbox_set_replay": (_ST, [vp, C.c_int]),
        "strassen_dist_create_loopback": (_ST, [C.POINTER(vp), vp, vp, C.c_int, C.c_int, C.c_int]),
        "strassen_dist_destroy": (None, [vp]),
        "strassen_dist_gemm": (_ST, [vp, vp, C.c_int, C.c_int, _L, _L, _L, C.c_double, vp, _L, vp,
                                     _L, vp, _L, _L]),
        "strassen_dist_last_counts": (_ST, [vp, C.POINTER(_L), C.POINTER(_L)]),
        "strassen_dist_position": (_ST, [vp] + [C.POINTER(C.c_int)] * 5),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def _lib_or_none():
    return _LIB


def lib():
    """The loaded C-ABI library; raises if it has not been built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run paper_1605_01078_b200.build() "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        _LIB = _declare(C.CDLL(LIB_PATH))
    return _LIB


def _check(status, what):
    if status != OK:
        raise StrassenError(status, what)


# ----------------------------------------------------------------- operands
def _operand(x):
    """(pointer, rows, cols, rs, cs, is_cuda) for a 2-D numpy array or torch tensor."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.dtype != torch.float64 or x.dim() != 2:
                raise TypeError("operands must be 2-D float64 tensors")
            return (x.data_ptr(), x.shape[0], x.shape[1], x.stride(0), x.stride(1), x.is_cuda)
    except ImportError:
        pass
    import numpy as np
    if isinstance(x, np.ndarray):
        if x.dtype != np.float64 or x.ndim != 2:
            raise TypeError("operands must be 2-D float64 arrays")
        return (x.ctypes.data, x.shape[0], x.shape[1], x.strides[0] // 8, x.strides[1] // 8, False)
    raise TypeError(f"unsupported operand type {type(x)!r}")


def _variant(v):
    return VARIANT_NAMES[v] if isinstance(v, str) else int(v)


class Ctx:
    """Opaque execution context (reference capi.cpp:12-18) plus device state."""

    def __init__(self):
        self._l = lib()
        self.ptr = C.c_void_p()
        _check(self._l.strassen_ctx_create(C.byref(self.ptr)), "ctx_create")

    def close(self):
        if self.ptr:
            self._l.strassen_ctx_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def blocking(self):
        b = Blocking()
        _check(self._l.strassen_ctx_get_blocking(self.ptr, C.byref(b)), "ctx_get_blocking")
        return {f: getattr(b, f) for f, _ in Blocking._fields_}

    def set_blocking(self, mc, nc, kc, mr, nr):
        _check(self._l.strassen_ctx_set_blocking(self.ptr, C.byref(Blocking(mc, nc, kc, mr, nr))),
               "ctx_set_blocking")

    def set_threads(self, t):
        _check(self._l.strassen_ctx_set_threads(self.ptr, int(t)), "ctx_set_threads")

    def enable_counters(self, on=True):
        _check(self._l.strassen_ctx_enable_counters(self.ptr, int(bool(on))), "enable_counters")

    def reset_counters(self):
        _check(self._l.strassen_ctx_reset_counters(self.ptr), "reset_counters")

    def counters(self):
        c = Counters()
        _check(self._l.strassen_ctx_get_counters(self.ptr, C.byref(c)), "get_counters")
        return {f: getattr(c, f) for f in COUNTER_FIELDS}

    def set_stream(self, stream):
        """cudaStream_t (int handle, torch.cuda.Stream or None)."""
        h = getattr(stream, "cuda_stream", stream)
        _check(self._l.strassen_ctx_set_stream(self.ptr, C.c_void_p(h or 0)), "set_stream")

    def last_launches(self):
        n = C.c_long()
        _check(self._l.strassen_ctx_last_launches(self.ptr, C.byref(n)), "last_launches")
        return n.value

    def set_peeling(self, on=True):
        """Odd fringes: dynamic peeling (default) or the reference's zero padding."""
        _check(self._l.strassen_ctx_set_peeling(self.ptr, int(bool(on))), "set_peeling")

    def set_pipelining(self, on=True):
        """Host calls: column-window pipelining of transfers and kernels (default on)."""
        _check(self._l.strassen_ctx_set_pipelining(self.ptr, int(bool(on))), "set_pipelining")

    def set_operand_events(self, a=None, b=None, c=None):
        """torch.cuda.Event (or None) per operand: the next call's kernels wait on it
        right before first reading that device operand."""
        h = [C.c_void_p(e.cuda_event if e is not None else None) for e in (a, b, c)]
        _check(self._l.strassen_ctx_set_operand_events(self.ptr, *h), "set_operand_events")

    def set_fused_terms(self, max_terms):
        """ABC / AB: operand sides of up to max_terms terms summed in the kernel,
        longer ones materialised first (bitwise-identical results)."""
        _check(self._l.strassen_ctx_set_fused_terms(self.ptr, int(max_terms)), "set_fused_terms")

    def set_max_level(self, level):
        """2 (default) or 3: level 3 for the naive / c variants (B200 extension)."""
        _check(self._l.strassen_ctx_set_max_level(self.ptr, int(level)), "set_max_level")

    def select(self, m, n, k):
        """(variant, level, predicted seconds) over the levels this ctx admits."""
        v, lv, t = C.c_int(), C.c_int(), C.c_double()
        _check(self._l.strassen_ctx_select(self.ptr, m, n, k, C.byref(v), C.byref(lv),
                                           C.byref(t)), "ctx_select")
        name = {val: key for key, val in VARIANT_NAMES.items()}[v.value]
        return name, lv.value, t.value

    def enable_profiling(self, on=True):
        _check(self._l.strassen_ctx_enable_profiling(self.ptr, int(bool(on))), "enable_profiling")

    def last_profile(self):
        """[{'kernel': name, 'ms': t}, ...] for the last compute call (profiling on)."""
        import json
        buf = C.create_string_buffer(1 << 16)
        _check(self._l.strassen_ctx_last_profile(self.ptr, buf, len(buf)), "last_profile")
        return json.loads(buf.value.decode())

    def workspace_bytes(self):
        n = C.c_long()
        _check(self._l.strassen_ctx_workspace_bytes(self.ptr, C.byref(n)), "workspace_bytes")
        return n.value

    # -------------------------------------------------------------- compute
    def gemm(self, variant, level, alpha, a, b, c):
        """C := alpha A B + C (reference strassen_gemm, strassen.h:82-86). Synchronous."""
        pa, m, k, rsa, csa, _ = _operand(a)
        pb, k2, n, rsb, csb, _ = _operand(b)
        pc, m2, n2, rsc, csc, _ = _operand(c)
        if k2 != k or m2 != m or n2 != n:
            raise ValueError("operand shapes mismatch")
        st = self._l.strassen_gemm(self.ptr, _variant(variant), int(level), m, n, k, float(alpha),
                                   C.c_void_p(pa), rsa, csa, C.c_void_p(pb), rsb, csb,
                                   C.c_void_p(pc), rsc, csc)
        _check(st, "strassen_gemm")
        return c

    def gemm_raw(self, variant, level, m, n, k, alpha, a, rsa, csa, b, rsb, csb, c, rsc, csc):
        """Unchecked ABI call with raw pointers; returns the status code."""
        return self._l.strassen_gemm(self.ptr, _variant(variant), int(level), m, n, k,
                                     float(alpha), a, rsa, csa, b, rsb, csb, c, rsc, csc)

    def gemm_device(self, variant, level, alpha, a, b, c, stream=None):
        """Asynchronous device entry (CUDA tensors, stream-ordered)."""
        pa, m, k, rsa, csa, ca = _operand(a)
        pb, k2, n, rsb, csb, cb = _operand(b)
        pc, m2, n2, rsc, csc, cc = _operand(c)
        if k2 != k or m2 != m or n2 != n:
            raise ValueError("operand shapes mismatch")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream()
        h = getattr(stream, "cuda_stream", stream)
        st = self._l.strassen_gemm_device(self.ptr, C.c_void_p(h), _variant(variant), int(level),
                                          m, n, k, float(alpha), C.c_void_p(pa), rsa, csa,
                                          C.c_void_p(pb), rsb, csb, C.c_void_p(pc), rsc, csc)
        _check(st, "strassen_gemm_device")
        return c

    def dgemm(self, variant, level, transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc):
        """Column-major BLAS-style shim with beta (raw pointers or arrays)."""
        def ptr(x):
            return C.c_void_p(x) if isinstance(x, int) else C.c_void_p(_operand(x)[0])
        st = self._l.strassen_dgemm(self.ptr, _variant(variant), int(level),
                                    transa.encode() if isinstance(transa, str) else transa,
                                    transb.encode() if isinstance(transb, str) else transb,
                                    m, n, k, float(alpha), ptr(a), lda, ptr(b), ldb, float(beta),
                                    ptr(c), ldc)
        _check(st, "strassen_dgemm")


_DEFAULT_CTX = None


def _ctx():
    global _DEFAULT_CTX
    if _DEFAULT_CTX is None:
        _DEFAULT_CTX = Ctx()
    return _DEFAULT_CTX


def gemm(variant, level, alpha, a, b, c, ctx=None):
    return (ctx or _ctx()).gemm(variant, level, alpha, a, b, c)


def gemm_device(variant, level, alpha, a, b, c, stream=None, ctx=None):
    return (ctx or _ctx()).gemm_device(variant, level, alpha, a, b, c, stream)


def dgemm(variant, level, transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, ctx=None):
    return (ctx or _ctx()).dgemm(variant, level, transa, transb, m, n, k, alpha, a, lda, b, ldb,
                                 beta, c, ldc)


def reference_gemm(alpha, a, b, c):
    """Host triple-loop reference product of the ABI (strassen_reference_gemm)."""
    pa, m, k, rsa, csa, _ = _operand(a)
    pb, _, n, rsb, csb, _ = _operand(b)
    pc, _, _, rsc, csc, _ = _operand(c)
    _check(lib().strassen_reference_gemm(m, n, k, float(alpha), C.c_void_p(pa), rsa, csa,
                                         C.c_void_p(pb), rsb, csb, C.c_void_p(pc), rsc, csc),
           "reference_gemm")
    return c


def rel_error(c_test, c_ref):
    pt, r, cc, rst, cst, _ = _operand(c_test)
    pr, _, _, rsr, csr, _ = _operand(c_ref)
    out = C.c_double()
    _check(lib().strassen_rel_error(r, cc, C.c_void_p(pt), rst, cst, C.c_void_p(pr), rsr, csr,
                                    C.byref(out)), "rel_error")
    return out.value


def table_counts(level):
    out = (C.c_long * 4)()
    _check(lib().strassen_table_counts(int(level), out), "table_counts")
    return tuple(out)


def effective_gflops(m, n, k, seconds):
    out = C.c_double()
    _check(lib().strassen_effective_gflops(m, n, k, float(seconds), C.byref(out)),
           "effective_gflops")
    return out.value


def blocking_defaults():
    b = Blocking()
    lib().strassen_blocking_defaults(C.byref(b))
    return {f: getattr(b, f) for f, _ in Blocking._fields_}


def model_params_ivy_bridge():
    p = ModelParams()
    lib().strassen_model_params_ivy_bridge(C.byref(p))
    return p


def model_predict(variant, level, m, n, k, blocking=None, params=None):
    bp = Blocking(**(blocking or blocking_defaults()))
    mp = params or model_params_ivy_bridge()
    bd = Breakdown()
    egf = C.c_double()
    _check(lib().strassen_model_predict(_variant(variant), int(level), m, n, k, C.byref(bp),
                                        C.byref(mp), C.byref(bd), C.byref(egf)), "model_predict")
    return {f: getattr(bd, f) for f, _ in Breakdown._fields_}, egf.value


def predicted_counters(variant, level, m, n, k, blocking=None):
    """Counter values one strassen_gemm call adds (analytic; no device needed)."""
    bp = Blocking(**(blocking or blocking_defaults()))
    c = Counters()
    _check(lib().strassen_count_call(_variant(variant), int(level), m, n, k, C.byref(bp),
                                     C.byref(c)), "count_call")
    return {f: getattr(c, f) for f in COUNTER_FIELDS}


def predict_b200(variant, level, m, n, k):
    """The B200 cost model's predicted seconds for one configuration."""
    t = C.c_double()
    _check(lib().strassen_predict_b200(_variant(variant), level, m, n, k, C.byref(t)),
           "predict_b200")
    return t.value


def select(m, n, k):
    """(variant name, level, predicted seconds) the B200 cost model picks for a shape."""
    v, lv, t = C.c_int(), C.c_int(), C.c_double()
    _check(lib().strassen_select(m, n, k, C.byref(v), C.byref(lv), C.byref(t)), "select")
    name = {val: key for key, val in VARIANT_NAMES.items()}[v.value]
    return name, lv.value, t.value
