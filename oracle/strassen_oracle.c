/*
 * strassen_oracle.c -- CPU restatement of the reference Strassen DGEMM path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * implementation.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product library
 * (paper_1605_01078_b200/) never links or calls it.
 *
 * It restates, in plain C, the algorithm of the reference
 * (/root/reference/proj/src, "Strassen's Algorithm Reloaded", arXiv 1605.01078)
 * with the SAME order of floating-point operations, so that its output is
 * bitwise identical to the reference library compiled with the reference's
 * own flags (-O3 -DNDEBUG, no -march; see oracle/Makefile).  That identity is
 * checked by tests/test_oracle.py against oracle/_ref/libstrassen_ref.so (the
 * reference itself, compiled from its own sources) and against the committed
 * golden vectors in tests/golden/ -- the oracle is "parity pinned".
 *
 * Restated pieces (reference file:line):
 *   so_mt19937_64 / so_fill_uniform    test_strassen.cpp:11-17, bench_lib.cpp:29-33
 *                                      (std::mt19937_64 + libstdc++
 *                                      uniform_real_distribution<double>)
 *   so_reference_gemm                  matrix.cpp:37-52 (triple loop, p ascending)
 *   so_rel_frobenius_error             matrix.cpp:54-66
 *   so_table                           table.cpp:14-35 (one level), :39-93 (compose)
 *   so_strassen_gemm                   variants.cpp:122-231 (ABC / AB / Naive /
 *                                      Dgemm), blocking.cpp:12-146 (packing sums,
 *                                      five-loop kc blocking), kernel.cpp:8-102
 *                                      (tile accumulate, multi-destination update)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SO_OK 0
#define SO_ERR_PARAM 2
#define SO_ERR_ALLOC 4

/* ---------------------------------------------------------------- RNG ---- */
/* std::mt19937_64 (the 64-bit Mersenne twister, MT19937-64 parameters). */
typedef struct {
    uint64_t mt[312];
    int idx;
} so_mt64;

static void mt64_seed(so_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(so_mt64* s) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    static const uint64_t MATA = 0xB5026F5AA96619E9ULL;
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= MATA;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* libstdc++ generate_canonical<double, 53> with a 64-bit engine: one draw,
 * sum = double(x) * 1, tmp = 2^64, ret = sum / tmp, clamped below 1. */
static double canonical(so_mt64* s) {
    const double r = 18446744073709551616.0; /* 2^64 */
    double ret = (double)mt64_next(s) / r;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}

/* uniform_real_distribution<double>(lo, hi): canonical * (hi - lo) + lo. */
void so_fill_uniform(double* p, long n, uint64_t seed, double lo, double hi) {
    so_mt64 s;
    mt64_seed(&s, seed);
    for (long i = 0; i < n; ++i) p[i] = canonical(&s) * (hi - lo) + lo;
}

/* Raw engine output, for pinning the generator against std::mt19937_64. */
void so_mt19937_64(uint64_t seed, long n, uint64_t* out) {
    so_mt64 s;
    mt64_seed(&s, seed);
    for (long i = 0; i < n; ++i) out[i] = mt64_next(&s);
}

/* ------------------------------------------------------------ oracle ---- */
/* matrix.cpp:37-52: row buffer keeps p ascending per (i, j). */
int so_reference_gemm(long m, long n, long k, double alpha, const double* a, long rsa,
                      long csa, const double* b, long rsb, long csb, double* c, long rsc,
                      long csc) {
    if (m < 1 || n < 1 || k < 1) return SO_ERR_PARAM;
    double* acc = (double*)malloc(sizeof(double) * (size_t)n);
    if (!acc) return SO_ERR_ALLOC;
    for (long i = 0; i < m; ++i) {
        for (long j = 0; j < n; ++j) acc[j] = 0.0;
        for (long p = 0; p < k; ++p) {
            const double av = a[i * rsa + p * csa];
            for (long j = 0; j < n; ++j) acc[j] += av * b[p * rsb + j * csb];
        }
        for (long j = 0; j < n; ++j) c[i * rsc + j * csc] += alpha * acc[j];
    }
    free(acc);
    return SO_OK;
}

/* matrix.cpp:54-66: ||T - R||_F / max(||R||_F, 1). */
double so_rel_frobenius_error(long rows, long cols, const double* t, long rst, long cst,
                              const double* r, long rsr, long csr) {
    double diff2 = 0.0, ref2 = 0.0;
    for (long i = 0; i < rows; ++i)
        for (long j = 0; j < cols; ++j) {
            const double d = t[i * rst + j * cst] - r[i * rsr + j * csr];
            diff2 += d * d;
            ref2 += r[i * rsr + j * csr] * r[i * rsr + j * csr];
        }
    const double den = sqrt(ref2) > 1.0 ? sqrt(ref2) : 1.0;
    return sqrt(diff2) / den;
}

/* BASELINE.json tolerance metric: ||dC||_F / (||A||_F * ||B||_F). */
double so_normwise_error(long m, long n, long k, const double* dc_t, const double* dc_r,
                         const double* a, const double* b) {
    /* dc_t / dc_r: dense m*n arrays (any consistent layout); a: m*k; b: k*n */
    long double d2 = 0, a2 = 0, b2 = 0;
    for (long i = 0; i < m * n; ++i) {
        long double d = (long double)dc_t[i] - (long double)dc_r[i];
        d2 += d * d;
    }
    for (long i = 0; i < m * k; ++i) a2 += (long double)a[i] * a[i];
    for (long i = 0; i < k * n; ++i) b2 += (long double)b[i] * b[i];
    if (a2 == 0 || b2 == 0) return (double)sqrtl(d2);
    return (double)(sqrtl(d2) / (sqrtl(a2) * sqrtl(b2)));
}

/* ------------------------------------------------------------- tables ---- */
/* One entry: up to 8 terms per side (level 3 composes to 8). */
#define SO_MAXT 8
typedef struct {
    int na, nb, nc;
    int aq[SO_MAXT], as[SO_MAXT];
    int bq[SO_MAXT], bs[SO_MAXT];
    int cq[SO_MAXT], cs[SO_MAXT];
} so_entry;

/* table.cpp:18-33, quadrant index = 2*row + col. */
static const int ONE[7][3][5] = {
    /* {count, q0, s0, q1, s1} for a, b, c */
    {{2, 0, 1, 3, 1}, {2, 0, 1, 3, 1}, {2, 0, 1, 3, 1}},
    {{2, 2, 1, 3, 1}, {1, 0, 1, 0, 0}, {2, 2, 1, 3, -1}},
    {{1, 0, 1, 0, 0}, {2, 1, 1, 3, -1}, {2, 1, 1, 3, 1}},
    {{1, 3, 1, 0, 0}, {2, 2, 1, 0, -1}, {2, 0, 1, 2, 1}},
    {{2, 0, 1, 1, 1}, {1, 3, 1, 0, 0}, {2, 1, 1, 0, -1}},
    {{2, 2, 1, 0, -1}, {2, 0, 1, 1, 1}, {1, 3, 1, 0, 0}},
    {{2, 1, 1, 3, -1}, {2, 2, 1, 3, 1}, {1, 0, 1, 0, 0}},
};

static void one_level(so_entry* t) {
    for (int e = 0; e < 7; ++e) {
        int* nn[3] = {&t[e].na, &t[e].nb, &t[e].nc};
        int* qq[3] = {t[e].aq, t[e].bq, t[e].cq};
        int* ss[3] = {t[e].as, t[e].bs, t[e].cs};
        for (int side = 0; side < 3; ++side) {
            *nn[side] = ONE[e][side][0];
            for (int u = 0; u < ONE[e][side][0]; ++u) {
                qq[side][u] = ONE[e][side][1 + 2 * u];
                ss[side][u] = ONE[e][side][2 + 2 * u];
            }
        }
    }
}

/* table.cpp:39-71: outer-term-major, duplicates merged, zeros dropped. */
static int compose_terms(int no, const int* oq, const int* os, int ni, const int* iq,
                         const int* is, int lo, int li, int* outq, int* outs) {
    const long so = 1L << lo, si = 1L << li, s = so * si;
    int n = 0;
    for (int a = 0; a < no; ++a) {
        const long orow = oq[a] / so, ocol = oq[a] % so;
        for (int b = 0; b < ni; ++b) {
            const long irow = iq[b] / si, icol = iq[b] % si;
            const int idx = (int)((si * orow + irow) * s + (si * ocol + icol));
            const int coeff = os[a] * is[b];
            int merged = 0;
            for (int u = 0; u < n; ++u)
                if (outq[u] == idx) {
                    outs[u] += coeff;
                    if (outs[u] < -1 || outs[u] > 1) return -1;
                    merged = 1;
                    break;
                }
            if (!merged) {
                if (n >= SO_MAXT) return -1;
                outq[n] = idx;
                outs[n] = coeff;
                ++n;
            }
        }
    }
    int w = 0; /* erase_if zero coefficient, order preserved */
    for (int u = 0; u < n; ++u)
        if (outs[u] != 0) {
            outq[w] = outq[u];
            outs[w] = outs[u];
            ++w;
        }
    return w;
}

/* table.cpp:75-93 / :95-102.  Returns number of entries (7^level), or -1.
 * Level 3 is built for symbolic checks (acceptance.cpp:86-88). */
int so_table(int level, so_entry* out) {
    if (level < 1 || level > 3) return -1;
    so_entry one[7];
    one_level(one);
    if (level == 1) {
        memcpy(out, one, sizeof(one));
        return 7;
    }
    so_entry prev[49];
    int nprev = 7, lprev = 1;
    memcpy(prev, one, sizeof(one));
    so_entry* cur = out;
    int n = 0;
    for (int L = 2; L <= level; ++L) {
        so_entry* dst = (L == level) ? cur : NULL;
        so_entry tmp[49];
        if (!dst) dst = tmp;
        n = 0;
        for (int e = 0; e < nprev; ++e)
            for (int f = 0; f < 7; ++f) {
                so_entry g;
                memset(&g, 0, sizeof(g));
                g.na = compose_terms(prev[e].na, prev[e].aq, prev[e].as, one[f].na, one[f].aq,
                                     one[f].as, lprev, 1, g.aq, g.as);
                g.nb = compose_terms(prev[e].nb, prev[e].bq, prev[e].bs, one[f].nb, one[f].bq,
                                     one[f].bs, lprev, 1, g.bq, g.bs);
                g.nc = compose_terms(prev[e].nc, prev[e].cq, prev[e].cs, one[f].nc, one[f].cq,
                                     one[f].cs, lprev, 1, g.cq, g.cs);
                if (g.na < 0 || g.nb < 0 || g.nc < 0) return -1;
                dst[n++] = g;
            }
        if (L < level) {
            memcpy(prev, dst, sizeof(so_entry) * (size_t)n);
            nprev = n;
            lprev = L;
        }
    }
    return n;
}

int so_entry_size(void) { return (int)sizeof(so_entry); }

/* ---------------------------------------------------------- variants ---- */
typedef struct {
    const double* p;
    long rows, cols, rs, cs;
} view_t;

/* matrix.cpp:8-35 (ceil rule, clipped, possibly empty views). */
static void partition(const double* base, long rows, long cols, long rs, long cs, int level,
                      view_t* v, long* qr, long* qc) {
    const long side = 1L << level;
    *qr = (rows + side - 1) / side;
    *qc = (cols + side - 1) / side;
    for (long I = 0; I < side; ++I)
        for (long J = 0; J < side; ++J) {
            const long r0 = I * *qr, c0 = J * *qc;
            long r = rows - r0 < *qr ? rows - r0 : *qr;
            long c = cols - c0 < *qc ? cols - c0 : *qc;
            if (r < 0) r = 0;
            if (c < 0) c = 0;
            view_t* w = &v[I * side + J];
            w->rows = r;
            w->cols = c;
            w->rs = rs;
            w->cs = cs;
            w->p = (r > 0 && c > 0) ? base + r0 * rs + c0 * cs : base;
        }
}

/* Operand sum of one (row, col) logical position, as pack_a_sum / pack_b_sum
 * build it (blocking.cpp:17-28): start from 0, add coeff * x in listed order,
 * skipping terms whose clipped view does not cover the position. */
static inline double term_sum(const view_t* v, const int* q, const int* s, int n, long i,
                              long j) {
    double acc = 0.0;
    for (int u = 0; u < n; ++u) {
        const view_t* w = &v[q[u]];
        if (i < w->rows && j < w->cols) acc += (double)s[u] * w->p[i * w->rs + j * w->cs];
    }
    return acc;
}

/*
 * One gemm_five_loop (blocking.cpp:82-131) over the logical qm x qn x qk
 * extent, restated without packing buffers but with the same arithmetic:
 * per kc block, T(i,j) = sum_p SA(i,p) * SB(p,j) from 0 with p ascending
 * (kernel.cpp:8-16), then for each destination in order
 * D(i,j) += (alpha * gamma) * T(i,j) for in-range (i, j) (kernel.cpp:49-76).
 * SA / SB are the packed operand sums.
 */
typedef struct {
    double* p;
    long rows, cols, rs, cs;
    int coeff;
} dest_t;

static int five_loop(long qm, long qn, long qk, double alpha, const view_t* av, const int* aq,
                     const int* as, int na, const view_t* bv, const int* bq, const int* bs,
                     int nb, const dest_t* d, int nd, long kc) {
    double* SA = (double*)malloc(sizeof(double) * (size_t)qm * (size_t)kc);
    double* SBt = (double*)malloc(sizeof(double) * (size_t)qn * (size_t)kc);
    if (!SA || !SBt) {
        free(SA);
        free(SBt);
        return SO_ERR_ALLOC;
    }
    for (long pc = 0; pc < qk; pc += kc) {
        const long k_c = (qk - pc < kc) ? qk - pc : kc;
        for (long i = 0; i < qm; ++i)
            for (long p = 0; p < k_c; ++p) SA[i * k_c + p] = term_sum(av, aq, as, na, i, pc + p);
        for (long j = 0; j < qn; ++j)
            for (long p = 0; p < k_c; ++p) SBt[j * k_c + p] = term_sum(bv, bq, bs, nb, pc + p, j);
#pragma omp parallel for schedule(static)
        for (long i = 0; i < qm; ++i) {
            int any_row = 0;
            for (int u = 0; u < nd; ++u)
                if (i < d[u].rows) any_row = 1;
            if (!any_row) continue;
            const double* ar = SA + i * k_c;
            for (long j = 0; j < qn; ++j) {
                const double* br = SBt + j * k_c;
                double t = 0.0;
                for (long p = 0; p < k_c; ++p) t += ar[p] * br[p];
                for (int u = 0; u < nd; ++u) {
                    if (i < d[u].rows && j < d[u].cols) {
                        const double s = alpha * (double)d[u].coeff;
                        d[u].p[i * d[u].rs + j * d[u].cs] += s * t;
                    }
                }
            }
        }
    }
    free(SA);
    free(SBt);
    return SO_OK;
}

static int all_empty(const view_t* v, const int* q, int n) {
    for (int u = 0; u < n; ++u)
        if (v[q[u]].rows > 0 && v[q[u]].cols > 0) return 0;
    return 1;
}

/* variants.cpp:53-96: materialize sum delta_s X_s into a zero-padded
 * rows x cols row-major temporary; first pass writes term 0 (or terms 0 and 1
 * in one expression), further terms accumulate. */
static void materialize(const view_t* v, const int* q, const int* s, int n, long rows,
                        long cols, double* buf) {
#define RD(w, i, j) (((i) < (w)->rows && (j) < (w)->cols) ? (w)->p[(i) * (w)->rs + (j) * (w)->cs] : 0.0)
    const view_t* x0 = &v[q[0]];
    const double d0 = s[0];
    int u = 1;
    if (n == 1) {
        for (long i = 0; i < rows; ++i)
            for (long j = 0; j < cols; ++j) buf[i * cols + j] = d0 * RD(x0, i, j);
    } else {
        const view_t* x1 = &v[q[1]];
        const double d1 = s[1];
        for (long i = 0; i < rows; ++i)
            for (long j = 0; j < cols; ++j)
                buf[i * cols + j] = d0 * RD(x0, i, j) + d1 * RD(x1, i, j);
        u = 2;
    }
    for (; u < n; ++u) {
        const view_t* xs = &v[q[u]];
        const double ds = s[u];
        for (long i = 0; i < rows; ++i)
            for (long j = 0; j < cols; ++j) buf[i * cols + j] += ds * RD(xs, i, j);
    }
#undef RD
}

/*
 * so_strassen_gemm: C := alpha A B + C.
 * variant: 0 = Dgemm (level must be 0), 1 = ABC, 2 = AB, 3 = Naive (level 1|2).
 * kc: the reference blocking kc (default 256, kernel.hpp:11-17); the other
 * blocking parameters do not change the arithmetic.
 */
int so_strassen_gemm(int variant, int level, long m, long n, long k, double alpha,
                     const double* a, long rsa, long csa, const double* b, long rsb, long csb,
                     double* c, long rsc, long csc, long kc) {
    if (m < 1 || n < 1 || k < 1 || kc < 1) return SO_ERR_PARAM;
    if (variant == 0) {
        if (level != 0) return SO_ERR_PARAM;
        view_t A = {a, m, k, rsa, csa}, B = {b, k, n, rsb, csb};
        const int q0 = 0, s1 = 1;
        dest_t D = {c, m, n, rsc, csc, 1};
        return five_loop(m, n, k, alpha, &A, &q0, &s1, 1, &B, &q0, &s1, 1, &D, 1, kc);
    }
    if (variant < 1 || variant > 3 || level < 1 || level > 2) return SO_ERR_PARAM;
    so_entry tab[49];
    const int ne = so_table(level, tab);
    view_t av[16], bv[16], cv[16];
    long qm, qk, qk2, qn, qm2, qn2;
    partition(a, m, k, rsa, csa, level, av, &qm, &qk);
    partition(b, k, n, rsb, csb, level, bv, &qk2, &qn);
    partition(c, m, n, rsc, csc, level, cv, &qm2, &qn2);
    double *M = NULL, *TA = NULL, *TB = NULL;
    if (variant >= 2) {
        M = (double*)malloc(sizeof(double) * (size_t)qm * (size_t)qn);
        if (!M) return SO_ERR_ALLOC;
    }
    if (variant == 3) {
        TA = (double*)malloc(sizeof(double) * (size_t)qm * (size_t)qk);
        TB = (double*)malloc(sizeof(double) * (size_t)qk * (size_t)qn);
        if (!TA || !TB) {
            free(M);
            free(TA);
            free(TB);
            return SO_ERR_ALLOC;
        }
    }
    int rc = SO_OK;
    for (int e = 0; e < ne && rc == SO_OK; ++e) {
        const so_entry* t = &tab[e];
        if (all_empty(av, t->aq, t->na) || all_empty(bv, t->bq, t->nb) ||
            all_empty(cv, t->cq, t->nc))
            continue;
        if (variant == 1) { /* variants.cpp:122-140 */
            dest_t d[SO_MAXT];
            for (int u = 0; u < t->nc; ++u) {
                const view_t* w = &cv[t->cq[u]];
                d[u].p = (double*)w->p;
                d[u].rows = w->rows;
                d[u].cols = w->cols;
                d[u].rs = w->rs;
                d[u].cs = w->cs;
                d[u].coeff = t->cs[u];
            }
            rc = five_loop(qm, qn, qk, alpha, av, t->aq, t->as, t->na, bv, t->bq, t->bs, t->nb,
                           d, t->nc, kc);
            continue;
        }
        /* AB / Naive (variants.cpp:142-208): M := 0; M += 1.0 * T; stream. */
        memset(M, 0, sizeof(double) * (size_t)qm * (size_t)qn);
        dest_t md = {M, qm, qn, qn, 1, 1};
        if (variant == 2) {
            rc = five_loop(qm, qn, qk, 1.0, av, t->aq, t->as, t->na, bv, t->bq, t->bs, t->nb,
                           &md, 1, kc);
        } else {
            materialize(av, t->aq, t->as, t->na, qm, qk, TA);
            materialize(bv, t->bq, t->bs, t->nb, qk, qn, TB);
            view_t ta = {TA, qm, qk, qk, 1}, tb = {TB, qk, qn, qn, 1};
            const int q0 = 0, s1 = 1;
            rc = five_loop(qm, qn, qk, 1.0, &ta, &q0, &s1, 1, &tb, &q0, &s1, 1, &md, 1, kc);
        }
        for (int u = 0; u < t->nc && rc == SO_OK; ++u) { /* variants.cpp:99-109 */
            const view_t* w = &cv[t->cq[u]];
            if (w->rows <= 0 || w->cols <= 0) continue;
            const double s = alpha * (double)t->cs[u];
            double* cp = (double*)w->p;
            for (long i = 0; i < w->rows; ++i)
                for (long j = 0; j < w->cols; ++j) cp[i * w->rs + j * w->cs] += s * M[i * qn + j];
        }
    }
    free(M);
    free(TA);
    free(TB);
    return rc;
}
