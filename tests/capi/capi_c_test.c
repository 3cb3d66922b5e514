/* Drop-in proof in plain C: a caller of the reference's C ABI, compiled against
 * include/strassen.h and linked to libstrassen_b200.so only (plus the oracle's
 * RNG, test infrastructure).  It ports, check for check:
 *   - the reference's C-API test suite, proj/tests/test_capi.cpp:27-185
 *     (lifecycle and blocking round trip, null / argument errors, the 117x93x201
 *     oracle match at alpha = 0.5 for all seven configurations, transposition by
 *     swapped strides, counters, model prediction, table counts and status strings);
 *   - the reference bench's call pattern, proj/tools/bench_lib.cpp:56-71 (run_once:
 *     the one-shot call and the rank-b schedule of repeated strassen_gemm calls on
 *     row-major buffers) and its verification, bench_lib.cpp:208-269
 *     (rel_frobenius against strassen_reference_gemm up to 1200, against
 *     STRASSEN_DGEMM above), emitting the reference CSV schema
 *     (bench_lib.cpp:138-157) with egf_modeled from strassen_model_predict.
 * Usage: capi_c_test [--no-device]   (--no-device: only the checks that make no
 * compute call; every compute call needs a CUDA device -- there is no CPU path). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "strassen.h"

/* test infrastructure: std::mt19937_64 + uniform_real_distribution(lo, hi), the
 * oracle's restatement (oracle/strassen_oracle.c), as test_capi.cpp:11-17 uses */
void so_fill_uniform(double* p, long n, uint64_t seed, double lo, double hi);

static int checks = 0, failures = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        ++checks;                                                              \
        if (!(cond)) {                                                         \
            ++failures;                                                        \
            fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
        }                                                                      \
    } while (0)
#define REQUIRE(cond)                                                          \
    do {                                                                       \
        ++checks;                                                              \
        if (!(cond)) {                                                         \
            fprintf(stderr, "FATAL %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
            exit(2);                                                           \
        }                                                                      \
    } while (0)

static double* random_vec(long n, uint64_t seed) {
    double* v = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    so_fill_uniform(v, n, seed, -1.0, 1.0);
    return v;
}

static double* copy_vec(const double* x, long n) {
    double* v = malloc(sizeof(double) * (size_t)n);
    memcpy(v, x, sizeof(double) * (size_t)n);
    return v;
}

/* test_capi.cpp:27-44 */
static void test_lifecycle_and_blocking(void) {
    strassen_ctx* ctx = NULL;
    REQUIRE(strassen_ctx_create(&ctx) == STRASSEN_OK);
    strassen_blocking bp;
    REQUIRE(strassen_ctx_get_blocking(ctx, &bp) == STRASSEN_OK);
    CHECK(bp.mc == 96);
    CHECK(bp.nc == 4096);
    CHECK(bp.kc == 256);
    CHECK(bp.mr == 8);
    CHECK(bp.nr == 4);
    bp.mc = 64;
    REQUIRE(strassen_ctx_set_blocking(ctx, &bp) == STRASSEN_OK);
    strassen_blocking back;
    REQUIRE(strassen_ctx_get_blocking(ctx, &back) == STRASSEN_OK);
    CHECK(back.mc == 64);
    bp.mc = 90; /* not a multiple of mr */
    CHECK(strassen_ctx_set_blocking(ctx, &bp) == STRASSEN_ERR_PARAM);
    strassen_ctx_destroy(ctx);
}

/* test_capi.cpp:46-67 */
static void test_null_and_argument_errors(void) {
    CHECK(strassen_ctx_create(NULL) == STRASSEN_ERR_NULL);
    CHECK(strassen_ctx_set_threads(NULL, 2) == STRASSEN_ERR_NULL);
    strassen_ctx* ctx = NULL;
    REQUIRE(strassen_ctx_create(&ctx) == STRASSEN_OK);
    CHECK(strassen_ctx_set_threads(ctx, 0) == STRASSEN_ERR_PARAM);
    double a[4] = {0}, b[4] = {0}, c[4] = {0};
    /* level 1 with the dgemm variant is inconsistent */
    CHECK(strassen_gemm(ctx, STRASSEN_DGEMM, 1, 2, 2, 2, 1.0, a, 2, 1, b, 2, 1, c, 2, 1) ==
          STRASSEN_ERR_PARAM);
    /* level 3 unsupported (by default) */
    CHECK(strassen_gemm(ctx, STRASSEN_ABC, 3, 2, 2, 2, 1.0, a, 2, 1, b, 2, 1, c, 2, 1) ==
          STRASSEN_ERR_PARAM);
    /* non-positive dimension */
    CHECK(strassen_gemm(ctx, STRASSEN_ABC, 1, -2, 2, 2, 1.0, a, 2, 1, b, 2, 1, c, 2, 1) ==
          STRASSEN_ERR_PARAM);
    /* null operand */
    CHECK(strassen_gemm(ctx, STRASSEN_ABC, 1, 2, 2, 2, 1.0, NULL, 2, 1, b, 2, 1, c, 2, 1) ==
          STRASSEN_ERR_NULL);
    strassen_ctx_destroy(ctx);
}

/* test_capi.cpp:69-95 */
static void test_oracle_match(void) {
    strassen_ctx* ctx = NULL;
    REQUIRE(strassen_ctx_create(&ctx) == STRASSEN_OK);
    REQUIRE(strassen_ctx_set_threads(ctx, 2) == STRASSEN_OK);
    const long m = 117, n = 93, k = 201;
    double* a = random_vec(m * k, 1);
    double* b = random_vec(k * n, 2);
    double* c0 = random_vec(m * n, 3);
    double* c_ref = copy_vec(c0, m * n);
    REQUIRE(strassen_reference_gemm(m, n, k, 0.5, a, k, 1, b, n, 1, c_ref, n, 1) == STRASSEN_OK);
    const strassen_variant variants[] = {STRASSEN_DGEMM, STRASSEN_ABC, STRASSEN_AB,
                                         STRASSEN_NAIVE};
    for (int vi = 0; vi < 4; ++vi) {
        const strassen_variant v = variants[vi];
        for (int level = (v == STRASSEN_DGEMM ? 0 : 1); level <= (v == STRASSEN_DGEMM ? 0 : 2);
             ++level) {
            double* c = copy_vec(c0, m * n);
            REQUIRE(strassen_gemm(ctx, v, level, m, n, k, 0.5, a, k, 1, b, n, 1, c, n, 1) ==
                    STRASSEN_OK);
            double err = 1.0;
            REQUIRE(strassen_rel_error(m, n, c, n, 1, c_ref, n, 1, &err) == STRASSEN_OK);
            CHECK(err < 1e-11);
            free(c);
        }
    }
    free(a);
    free(b);
    free(c0);
    free(c_ref);
    strassen_ctx_destroy(ctx);
}

/* test_capi.cpp:97-115 */
static void test_transposition(void) {
    strassen_ctx* ctx = NULL;
    REQUIRE(strassen_ctx_create(&ctx) == STRASSEN_OK);
    const long m = 20, n = 15, k = 30;
    double* at = random_vec(k * m, 4); /* A stored transposed (k x m, row-major) */
    double* b = random_vec(k * n, 5);
    double* c = calloc((size_t)(m * n), sizeof(double));
    double* c_ref = calloc((size_t)(m * n), sizeof(double));
    REQUIRE(strassen_gemm(ctx, STRASSEN_ABC, 1, m, n, k, 1.0, at, 1, m, b, n, 1, c, n, 1) ==
            STRASSEN_OK);
    double* a = malloc(sizeof(double) * (size_t)(m * k));
    for (long i = 0; i < m; ++i)
        for (long p = 0; p < k; ++p) a[i * k + p] = at[p * m + i];
    REQUIRE(strassen_reference_gemm(m, n, k, 1.0, a, k, 1, b, n, 1, c_ref, n, 1) == STRASSEN_OK);
    double err = 1.0;
    REQUIRE(strassen_rel_error(m, n, c, n, 1, c_ref, n, 1, &err) == STRASSEN_OK);
    CHECK(err < 1e-12);
    free(at);
    free(b);
    free(c);
    free(c_ref);
    free(a);
    strassen_ctx_destroy(ctx);
}

/* test_capi.cpp:117-136 */
static void test_counters(void) {
    strassen_ctx* ctx = NULL;
    REQUIRE(strassen_ctx_create(&ctx) == STRASSEN_OK);
    REQUIRE(strassen_ctx_enable_counters(ctx, 1) == STRASSEN_OK);
    const long d = 64;
    double* a = random_vec(d * d, 6);
    double* b = random_vec(d * d, 7);
    double* c = calloc((size_t)(d * d), sizeof(double));
    REQUIRE(strassen_gemm(ctx, STRASSEN_NAIVE, 1, d, d, d, 1.0, a, d, 1, b, d, 1, c, d, 1) ==
            STRASSEN_OK);
    strassen_counter_values cv;
    REQUIRE(strassen_ctx_get_counters(ctx, &cv) == STRASSEN_OK);
    CHECK(cv.a_plus_passes == 19);
    CHECK(cv.b_plus_passes == 19);
    CHECK(cv.c_plus_passes == 36);
    CHECK(cv.kernel_fma_flops == 7 * 2 * 32 * 32 * 32);
    REQUIRE(strassen_ctx_reset_counters(ctx) == STRASSEN_OK);
    REQUIRE(strassen_ctx_get_counters(ctx, &cv) == STRASSEN_OK);
    CHECK(cv.a_plus_passes == 0);
    CHECK(cv.kernel_calls == 0);
    free(a);
    free(b);
    free(c);
    strassen_ctx_destroy(ctx);
}

/* test_capi.cpp:138-169 */
static void test_model(void) {
    strassen_blocking bp;
    strassen_blocking_defaults(&bp);
    strassen_model_params mp;
    strassen_model_params_ivy_bridge(&mp);
    CHECK(mp.lambda == 0.7);
    CHECK(mp.channel_factor == 4.0);
    strassen_breakdown bd;
    double egf = 0.0;
    REQUIRE(strassen_model_predict(STRASSEN_ABC, 1, 16000, 16000, 512, &bp, &mp, &bd, &egf) ==
            STRASSEN_OK);
    CHECK(bd.total == bd.ta_mul + bd.ta_a_add + bd.ta_b_add + bd.ta_c_add + bd.tm_a_mul +
                          bd.tm_b_mul + bd.tm_c_mul + bd.tm_a_add + bd.tm_b_add + bd.tm_c_add);
    CHECK(egf > 0.0);
    strassen_breakdown bd_dg;
    double egf_dg = 0.0;
    REQUIRE(strassen_model_predict(STRASSEN_DGEMM, 0, 16000, 16000, 512, &bp, &mp, &bd_dg,
                                   &egf_dg) == STRASSEN_OK);
    CHECK(bd.total < bd_dg.total);
    CHECK(strassen_model_predict(STRASSEN_ABC, 3, 100, 100, 100, &bp, &mp, &bd, &egf) ==
          STRASSEN_ERR_PARAM);
    double out = 0.0;
    CHECK(strassen_effective_gflops(10, 10, 10, 0.0, &out) == STRASSEN_ERR_DOMAIN);
    REQUIRE(strassen_effective_gflops(1000, 1000, 1000, 1.0, &out) == STRASSEN_OK);
    CHECK(out == 2.0);
}

/* test_capi.cpp:171-185 */
static void test_table_counts_and_status(void) {
    long c1[4] = {0, 0, 0, 0};
    REQUIRE(strassen_table_counts(1, c1) == STRASSEN_OK);
    CHECK(c1[0] == 7 && c1[1] == 5 && c1[2] == 5 && c1[3] == 12);
    long c2[4] = {0, 0, 0, 0};
    REQUIRE(strassen_table_counts(2, c2) == STRASSEN_OK);
    CHECK(c2[0] == 49 && c2[1] == 95 && c2[2] == 95 && c2[3] == 144);
    CHECK(strassen_table_counts(3, c2) == STRASSEN_ERR_PARAM);
    CHECK(strcmp(strassen_status_str(STRASSEN_OK), "ok") == 0);
    CHECK(strlen(strassen_status_str(STRASSEN_ERR_DIMENSION)) > 0);
}

/* ---- the reference bench's call pattern and verification ------------------ */
typedef struct {
    strassen_variant v;
    int level;
    const char* name;
} variant_config;

/* bench_lib.cpp:56-71: one multiplication; for rank-b the schedule of rank-b
 * updates C += A[:, p0:p0+b] B[p0:p0+b, :] on row-major buffers */
static strassen_status run_once(strassen_ctx* ctx, const variant_config* vc, long panel_b, long m,
                                long n, long k, const double* a, const double* b, double* c) {
    if (panel_b > 0) {
        for (long p0 = 0; p0 < k; p0 += panel_b) {
            const long bw = panel_b < k - p0 ? panel_b : k - p0;
            strassen_status s = strassen_gemm(ctx, vc->v, vc->level, m, n, bw, 1.0, a + p0, k, 1,
                                              b + p0 * n, n, 1, c, n, 1);
            if (s != STRASSEN_OK) return s;
        }
        return STRASSEN_OK;
    }
    return strassen_gemm(ctx, vc->v, vc->level, m, n, k, 1.0, a, k, 1, b, n, 1, c, n, 1);
}

/* bench_lib.cpp:80-96: modeled seconds, summed over the rank-b panels */
static double model_seconds(const variant_config* vc, long panel_b, long m, long n, long k) {
    strassen_blocking bp;
    strassen_blocking_defaults(&bp);
    strassen_model_params mp;
    strassen_model_params_ivy_bridge(&mp);
    const long step = panel_b > 0 ? panel_b : k;
    double total = 0.0;
    for (long p0 = 0; p0 < k; p0 += step) {
        const long bw = step < k - p0 ? step : k - p0;
        strassen_breakdown bd;
        if (strassen_model_predict(vc->v, vc->level, m, n, bw, &bp, &mp, &bd, NULL) != STRASSEN_OK)
            return -1.0;
        total += bd.total;
    }
    return total;
}

/* bench_lib.cpp:195-269 for one shape: seeds, oracle choice, one row per variant */
static void bench_shape(strassen_ctx* ctx, long m, long n, long k, long panel_b, FILE* csv) {
    const uint64_t seed = 0x9e3779b97f4a7c15ull ^ (uint64_t)m << 40 ^ (uint64_t)n << 20 ^ (uint64_t)k;
    double* a = random_vec(m * k, seed);
    double* b = random_vec(k * n, seed + 1);
    double* c0 = random_vec(m * n, seed + 2);
    double* c_ref = copy_vec(c0, m * n);
    if ((m > n ? (m > k ? m : k) : (n > k ? n : k)) <= 1200)
        REQUIRE(strassen_reference_gemm(m, n, k, 1.0, a, k, 1, b, n, 1, c_ref, n, 1) ==
                STRASSEN_OK);
    else
        REQUIRE(strassen_gemm(ctx, STRASSEN_DGEMM, 0, m, n, k, 1.0, a, k, 1, b, n, 1, c_ref, n,
                              1) == STRASSEN_OK);
    const variant_config vcs[] = {{STRASSEN_DGEMM, 0, "dgemm"}, {STRASSEN_ABC, 1, "abc"},
                                  {STRASSEN_AB, 1, "ab"},       {STRASSEN_NAIVE, 1, "naive"},
                                  {STRASSEN_ABC, 2, "abc"},     {STRASSEN_AB, 2, "ab"},
                                  {STRASSEN_NAIVE, 2, "naive"}};
    double* c = malloc(sizeof(double) * (size_t)(m * n));
    for (int i = 0; i < 7; ++i) {
        memcpy(c, c0, sizeof(double) * (size_t)(m * n));
        REQUIRE(run_once(ctx, &vcs[i], panel_b, m, n, k, a, b, c) == STRASSEN_OK);
        double err = 1.0;
        REQUIRE(strassen_rel_error(m, n, c, n, 1, c_ref, n, 1, &err) == STRASSEN_OK);
        CHECK(err < 1e-11); /* the reference bench's verify_tol default */
        double egf_modeled = 0.0;
        const double tm = model_seconds(&vcs[i], panel_b, m, n, k);
        CHECK(tm > 0.0 && strassen_effective_gflops(m, n, k, tm, &egf_modeled) == STRASSEN_OK);
        /* bench_lib.cpp:138-157 schema; time / egf_measured are the timing harness's */
        fprintf(csv, "%ld,%ld,%ld,%s,%d,1,1,,,%.17g,%.17g\n", m, n, k, vcs[i].name,
                vcs[i].level, egf_modeled, err);
    }
    free(a);
    free(b);
    free(c0);
    free(c_ref);
    free(c);
}

static void test_bench_call_pattern(void) {
    strassen_ctx* ctx = NULL;
    REQUIRE(strassen_ctx_create(&ctx) == STRASSEN_OK);
    printf("m,n,k,variant,level,threads,reps,time_s,egf_measured,egf_modeled,rel_err\n");
    bench_shape(ctx, 300, 257, 400, 0, stdout);     /* square-ish, reference_gemm oracle */
    bench_shape(ctx, 512, 512, 1024, 256, stdout);  /* rank-b schedule, b = 256 */
    bench_shape(ctx, 1300, 1290, 700, 0, stdout);   /* above 1200: the DGEMM oracle */
    strassen_ctx_destroy(ctx);
}

int main(int argc, char** argv) {
    const int device = !(argc > 1 && strcmp(argv[1], "--no-device") == 0);
    test_lifecycle_and_blocking();
    test_null_and_argument_errors();
    test_model();
    test_table_counts_and_status();
    if (device) {
        test_oracle_match();
        test_transposition();
        test_counters();
        test_bench_call_pattern();
    }
    printf("%s: %d checks, %d failures (%s)\n", failures ? "FAIL" : "PASS", checks, failures,
           device ? "device" : "no device");
    return failures ? 1 : 0;
}
