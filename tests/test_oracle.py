"""The parity checker itself: pinned against the reference's golden vectors
and known answers before anything is compared against it (CPU only)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle_lib as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))
GOLDEN_NPZ = np.load(os.path.join(HERE, "golden", "golden.npz"))


def golden_inputs(case):
    m, n, k = case["m"], case["n"], case["k"]
    s = case["seeds"]
    a, b, c = O.fill_uniform(m * k, s[0]), O.fill_uniform(k * n, s[1]), O.fill_uniform(m * n, s[2])
    if case["layout"] == "row":
        return a.reshape(m, k), b.reshape(k, n), c.reshape(m, n)
    return a.reshape(k, m).T, b.reshape(n, k).T, c.reshape(n, m).T


def test_mt19937_64_known_answer():
    # C++ [rand.predef]: the 10000th output of a default-constructed mt19937_64
    assert int(O.mt19937_64(5489, 10000)[-1]) == 9981545732273789042
    assert GOLDEN["mt19937_64_seed5489_10000th"] == 9981545732273789042


@pytest.mark.parametrize("case", GOLDEN["cases"], ids=lambda c: c["key"])
def test_oracle_reproduces_reference_golden(case):
    """Bitwise: the C restatement equals the reference's own outputs."""
    a, b, c = golden_inputs(case)
    c = c.copy(order="A")
    if case["variant"] == "reference":
        O.reference_gemm(case["alpha"], a, b, c)
    else:
        O.strassen_gemm(case["variant"], case["level"], case["alpha"], a, b, c)
    data = np.ascontiguousarray(c)
    assert hashlib.sha256(data.tobytes()).hexdigest() == case["sha256"]
    if case["full"]:
        assert np.array_equal(data, GOLDEN_NPZ[case["key"]])


def test_reference_gemm_known_answers():
    # test_matrix.cpp:39-45: [[1,2],[3,4]] [[5,6],[7,8]] = [[19,22],[43,50]]
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[5.0, 6.0], [7.0, 8.0]])
    c = np.zeros((2, 2))
    O.reference_gemm(1.0, a, b, c)
    assert np.array_equal(c, [[19.0, 22.0], [43.0, 50.0]])
    # identity and alpha = 0 (test_matrix.cpp:21-37)
    x = O.fill_uniform(25, 3).reshape(5, 5)
    c = np.zeros((5, 5))
    O.reference_gemm(1.0, np.eye(5), x, c)
    assert np.array_equal(c, x)
    c0 = O.fill_uniform(25, 4).reshape(5, 5)
    c = c0.copy()
    O.reference_gemm(0.0, x, x, c)
    assert np.array_equal(c, c0)


def test_seven_product_formula_bitwise():
    # test_strassen.cpp:31-62
    a = O.fill_uniform(4, 1).reshape(2, 2)
    b = O.fill_uniform(4, 2).reshape(2, 2)
    c = O.fill_uniform(4, 3).reshape(2, 2)
    want = c.copy()
    al = 0.5
    m0 = (a[0, 0] + a[1, 1]) * (b[0, 0] + b[1, 1])
    m1 = (a[1, 0] + a[1, 1]) * b[0, 0]
    m2 = a[0, 0] * (b[0, 1] - b[1, 1])
    m3 = a[1, 1] * (b[1, 0] - b[0, 0])
    m4 = (a[0, 0] + a[0, 1]) * b[1, 1]
    m5 = (a[1, 0] - a[0, 0]) * (b[0, 0] + b[0, 1])
    m6 = (a[0, 1] - a[1, 1]) * (b[1, 0] + b[1, 1])
    for (i, j), g, mv in [((0, 0), 1, m0), ((1, 1), 1, m0), ((1, 0), 1, m1), ((1, 1), -1, m1),
                          ((0, 1), 1, m2), ((1, 1), 1, m2), ((0, 0), 1, m3), ((1, 0), 1, m3),
                          ((0, 1), 1, m4), ((0, 0), -1, m4), ((1, 1), 1, m5), ((0, 0), 1, m6)]:
        want[i, j] += (al * g) * mv
    O.strassen_gemm("abc", 1, al, a, b, c)
    assert np.array_equal(c, want)


def _symbolic(table, level):
    s = 1 << level
    got = [dict() for _ in range(s * s)]
    for a_t, b_t, c_t in table:
        prod = {}
        for qa, da in a_t:
            for qb, eb in b_t:
                prod[(qa, qb)] = prod.get((qa, qb), 0) + da * eb
        for qc, g in c_t:
            for mono, co in prod.items():
                got[qc][mono] = got[qc].get(mono, 0) + g * co
    for p in got:
        for key in [k for k, v in p.items() if v == 0]:
            del p[key]
    for i in range(s):
        for j in range(s):
            want = {(i * s + p, p * s + j): 1 for p in range(s)}
            if got[i * s + j] != want:
                return False
    return True


@pytest.mark.parametrize("level", [1, 2, 3])
def test_tables_symbolically_correct(level):
    # symbolic_oracle.hpp:35-47; acceptance.cpp:82-89
    t = O.table(level)
    assert len(t) == 7 ** level
    assert _symbolic(t, level)


def test_table_golden_entries_and_counts():
    t1 = O.table(1)
    assert t1[2] == ([(0, 1)], [(1, 1), (3, -1)], [(1, 1), (3, 1)])      # test_table.cpp:32-35
    assert t1[5] == ([(2, 1), (0, -1)], [(0, 1), (1, 1)], [(3, 1)])      # :36-39
    assert t1[0] == ([(0, 1), (3, 1)], [(0, 1), (3, 1)], [(0, 1), (3, 1)])
    for L, want in [(1, (7, 5, 5, 12)), (2, (49, 95, 95, 144))]:
        t = O.table(L)
        counts = (len(t), sum(len(e[0]) - 1 for e in t), sum(len(e[1]) - 1 for e in t),
                  sum(len(e[2]) for e in t))
        assert counts == want
    t2 = O.table(2)
    assert t2[0] == ([(0, 1), (5, 1), (10, 1), (15, 1)],) * 3
    assert t2[48] == ([(3, 1), (7, -1), (11, -1), (15, 1)], [(12, 1), (13, 1), (14, 1), (15, 1)],
                      [(0, 1)])
    assert [[list(x) for x in side] for e in t2 for side in e] == \
        [side for e in GOLDEN["tables"]["2"] for side in e]


@pytest.mark.skipif(not O.RefStrassen.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_reference_library_random(seed):
    """Random shapes, strides and alphas: bitwise equality with the reference .so."""
    rng = np.random.default_rng(seed)
    ref = O.RefStrassen()
    m, n, k = (int(x) for x in rng.integers(1, 200, size=3))
    alpha = [1.0, -1.0, 0.5][seed % 3]
    a = O.fill_uniform(m * k, 10 + seed).reshape(m, k)
    b = O.fill_uniform(k * n, 20 + seed).reshape(k, n)
    c0 = O.fill_uniform(m * n, 30 + seed).reshape(m, n)
    if seed % 2:
        a, b = np.asfortranarray(a), np.asfortranarray(b)
    for v, L in [("dgemm", 0), ("abc", 1), ("ab", 1), ("naive", 1), ("abc", 2), ("ab", 2),
                 ("naive", 2)]:
        c1, c2 = c0.copy(), c0.copy()
        O.strassen_gemm(v, L, alpha, a, b, c1)
        ref.gemm(v, L, alpha, a, b, c2)
        assert np.array_equal(c1, c2), (v, L, m, n, k)


def test_error_metrics():
    x = O.fill_uniform(12, 5).reshape(3, 4)
    assert O.rel_frobenius_error(x, x) == 0.0
    z = np.zeros((3, 4))
    assert O.rel_frobenius_error(z + 0.5, z) == pytest.approx(np.sqrt(12 * 0.25))  # max(||R||,1)
    a = np.ones((3, 2))
    b = np.ones((2, 4))
    assert O.normwise_error(x, x, a, b) == 0.0
