"""Generate the committed golden vectors from the REFERENCE ITSELF.

Runs oracle/_ref/libstrassen_ref.so (the reference library compiled from
/root/reference/proj/src by oracle/Makefile) on seeded inputs and stores
  golden.npz  : full outputs for small shapes (bitwise)
  golden.json : case metadata + sha256 of the output bytes for every case
Inputs are regenerated at test time from the same seeds with
std::mt19937_64 + uniform_real_distribution<double>(-1, 1) (the reference's
test convention, test_strassen.cpp:11-17), via the oracle's pinned RNG.

Usage (in the build container, where the reference is present):
    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as O  # noqa: E402

CONFIGS = [("dgemm", 0), ("abc", 1), ("ab", 1), ("naive", 1), ("abc", 2), ("ab", 2), ("naive", 2)]
# (m, n, k, alpha, layout, seeds): shapes from the reference's own tests
# (test_matrix.cpp:39-45, test_strassen.cpp:84-100, test_capi.cpp:69-95) plus fringe cases.
CASES = [
    (2, 2, 2, 0.5, "row", (1, 2, 3)),
    (1, 1, 1, 1.0, "row", (101, 201, 301)),
    (3, 3, 3, 1.0, "row", (103, 203, 303)),
    (31, 79, 127, 1.0, "row", (131, 279, 427)),
    (129, 64, 5, 1.0, "row", (229, 264, 305)),
    (2, 300, 2, 1.0, "row", (102, 500, 302)),
    (33, 17, 65, -1.0, "col", (7, 8, 9)),
    (64, 64, 64, 1.0, "col", (6, 7, 0)),
    (117, 93, 201, 0.5, "row", (1, 2, 3)),
    (300, 290, 520, 1.0, "col", (11, 12, 13)),
]
FULL_LIMIT = 64 * 64  # store full outputs up to this many elements


def inputs(m, n, k, layout, seeds):
    a = O.fill_uniform(m * k, seeds[0])
    b = O.fill_uniform(k * n, seeds[1])
    c = O.fill_uniform(m * n, seeds[2])
    if layout == "row":
        return a.reshape(m, k), b.reshape(k, n), c.reshape(m, n)
    return (a.reshape(k, m).T, b.reshape(n, k).T, c.reshape(n, m).T)  # column-major views


def main():
    ref = O.RefStrassen()
    meta, arrays = [], {}
    for (m, n, k, alpha, layout, seeds) in CASES:
        a, b, c0 = inputs(m, n, k, layout, seeds)
        for v, lvl in CONFIGS:
            c = c0.copy(order="A")
            ref.gemm(v, lvl, alpha, a, b, c)
            key = f"{m}x{n}x{k}_{layout}_{v}{lvl}"
            data = np.ascontiguousarray(c).tobytes()
            meta.append(dict(key=key, m=m, n=n, k=k, alpha=alpha, layout=layout, seeds=seeds,
                             variant=v, level=lvl, sha256=hashlib.sha256(data).hexdigest(),
                             full=m * n <= FULL_LIMIT))
            if m * n <= FULL_LIMIT:
                arrays[key] = np.ascontiguousarray(c)
        # the triple-loop oracle too (matrix.cpp:37-52)
        c = c0.copy(order="A")
        ref.lib.strassen_reference_gemm(m, n, k, alpha, *O_ptrs(a, b, c))
        key = f"{m}x{n}x{k}_{layout}_reference"
        meta.append(dict(key=key, m=m, n=n, k=k, alpha=alpha, layout=layout, seeds=seeds,
                         variant="reference", level=0,
                         sha256=hashlib.sha256(np.ascontiguousarray(c).tobytes()).hexdigest(),
                         full=m * n <= FULL_LIMIT))
        if m * n <= FULL_LIMIT:
            arrays[key] = np.ascontiguousarray(c)
    tables = {str(L): O.table(L) for L in (1, 2)}
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(dict(generator="oracle/_ref/libstrassen_ref.so (reference compiled from its "
                       "own sources, -O3 -DNDEBUG -fopenmp)", cases=meta, tables=tables,
                       mt19937_64_seed5489_10000th=int(O.mt19937_64(5489, 10000)[-1])),
                  f, indent=1)
    print(f"wrote {len(meta)} cases, {len(arrays)} full arrays")


def O_ptrs(a, b, c):
    import ctypes as C
    dp = C.POINTER(C.c_double)
    s = lambda x: (x.strides[0] // 8, x.strides[1] // 8)  # noqa: E731
    return (a.ctypes.data_as(dp), *s(a), b.ctypes.data_as(dp), *s(b), c.ctypes.data_as(dp), *s(c))


if __name__ == "__main__":
    main()
