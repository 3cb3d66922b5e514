"""Correctness check of one variant through a minimal ctypes binding (works with older
library builds, for bisecting): check_variant.py lib.so m level variant reps.
Prints the number of 128x128 tiles off the cuBLAS result (> 1e-9) per run."""
import sys, ctypes as C
import torch
lib = C.CDLL(sys.argv[1])
m, L, v, reps = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
VAR = {"dgemm": 0, "abc": 1, "ab": 2, "naive": 3, "c": 4}[v]
ctx = C.c_void_p()
assert lib.strassen_ctx_create(C.byref(ctx)) == 0
f = lib.strassen_gemm_device
f.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_long, C.c_long, C.c_long, C.c_double,
              C.c_void_p, C.c_long, C.c_long, C.c_void_p, C.c_long, C.c_long, C.c_void_p, C.c_long, C.c_long]
g = torch.Generator(device="cuda").manual_seed(1)
A = (torch.rand(m, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
B = (torch.rand(m, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
C0 = (torch.rand(m, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
ref = C0 + A @ B
nbad = []
for r in range(reps):
    Cm = C0.clone().t().contiguous().t()
    st = f(ctx, None, VAR, L, m, m, m, 1.0, A.data_ptr(), 1, m, B.data_ptr(), 1, m, Cm.data_ptr(), 1, m)
    torch.cuda.synchronize()
    T = m // 128
    d = (Cm - ref).abs()
    nbad.append(int(((d.reshape(T, 128, T, 128).amax(dim=(1, 3))) > 1e-9).sum().item()))
print(sys.argv[1].split('/')[-1], v, L, m, "status", st, "bad tiles per run", nbad, flush=True)
