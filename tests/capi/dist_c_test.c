/* A plain-C caller of the native distributed entry points (include/strassen_dist.h),
 * compiled against the headers and linked to libstrassen_b200.so and the CUDA runtime.
 *
 *   dist_c_test --no-device        schedule functions and validation only
 *   dist_c_test                    + a 1 x 1 grid over NCCL on the visible GPU and a
 *                                    2 x 2 grid through the loopback transport, both
 *                                    checked against strassen_reference_gemm (the
 *                                    reference's oracle choice, bench_lib.cpp:210-214)
 *
 * A real multi-GPU caller does exactly what run_nccl() does with rank/nranks from its
 * launcher and the unique id handed round by its own means (MPI_Bcast, a file).
 */
#include <cuda_runtime_api.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "strassen.h"
#include "strassen_dist.h"

static int failures = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

static double urand(unsigned long long* s) { /* splitmix64 -> [-1, 1) */
    unsigned long long z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

static void schedule_checks(void) {
    int pr = 0, pc = 0;
    CHECK(strassen_dist_grid(1, &pr, &pc) == STRASSEN_OK && pr == 1 && pc == 1);
    CHECK(strassen_dist_grid(2, &pr, &pc) == STRASSEN_OK && pr == 1 && pc == 2);
    CHECK(strassen_dist_grid(4, &pr, &pc) == STRASSEN_OK && pr == 2 && pc == 2);
    CHECK(strassen_dist_grid(8, &pr, &pc) == STRASSEN_OK && pr == 2 && pc == 4);
    CHECK(strassen_dist_grid(0, &pr, &pc) == STRASSEN_ERR_PARAM);
    CHECK(strassen_dist_grid(8, NULL, &pc) == STRASSEN_ERR_NULL);
    CHECK(strassen_dist_default_panel(65536) == 8192);
    CHECK(strassen_dist_default_panel(1024) == 1024);

    strassen_dist_piece pieces[8];
    long count = 0;
    /* 2 x 4 grid, k = 48: A owners hold 12 columns, B owners 24 rows; panel 1 of width 24 */
    CHECK(strassen_dist_panel_pieces(48, 2, 4, 24, 1, 0, pieces, 8, &count) == STRASSEN_OK);
    CHECK(count == 2 && pieces[0].owner == 2 && pieces[0].local_off == 0 &&
          pieces[0].width == 12 && pieces[0].panel_off == 0 && pieces[1].owner == 3 &&
          pieces[1].panel_off == 12);
    CHECK(strassen_dist_panel_pieces(48, 2, 4, 24, 1, 1, pieces, 8, &count) == STRASSEN_OK);
    CHECK(count == 1 && pieces[0].owner == 1 && pieces[0].local_off == 0 && pieces[0].width == 24);
    CHECK(strassen_dist_panel_pieces(48, 2, 4, 5, 0, 0, pieces, 8, &count) == STRASSEN_ERR_PARAM);
    CHECK(strassen_dist_panel_pieces(48, 2, 4, 24, 2, 0, pieces, 8, &count) == STRASSEN_ERR_PARAM);
    CHECK(strassen_dist_panel_pieces(50, 2, 4, 25, 0, 0, pieces, 8, &count) == STRASSEN_ERR_PARAM);
    CHECK(strassen_dist_panel_pieces(48, 2, 4, 24, 0, 0, pieces, 8, NULL) == STRASSEN_ERR_NULL);

    strassen_dist* d = NULL;
    CHECK(strassen_dist_create(&d, NULL, "x", 0, 1, 1, 1) == STRASSEN_ERR_NULL);
    CHECK(strassen_dist_gemm(NULL, NULL, STRASSEN_ABC, 1, 8, 8, 8, 1.0, NULL, 8, NULL, 8, NULL, 8,
                             0) == STRASSEN_ERR_NULL);
}

/* Global column-major A (m x k), B (k x n), C (m x n) on the host; rank (i, j)'s blocks
 * are copied to the device with leading dimension ld* = rows + pad. */
typedef struct {
    long m, n, k;
    double *a, *b, *c, *want;
} Problem;

static Problem make_problem(long m, long n, long k, double alpha, unsigned long long seed) {
    Problem p = {m, n, k, NULL, NULL, NULL, NULL};
    p.a = malloc(sizeof(double) * m * k);
    p.b = malloc(sizeof(double) * k * n);
    p.c = malloc(sizeof(double) * m * n);
    p.want = malloc(sizeof(double) * m * n);
    for (long t = 0; t < m * k; ++t) p.a[t] = urand(&seed);
    for (long t = 0; t < k * n; ++t) p.b[t] = urand(&seed);
    for (long t = 0; t < m * n; ++t) p.c[t] = urand(&seed);
    memcpy(p.want, p.c, sizeof(double) * m * n);
    strassen_reference_gemm(m, n, k, alpha, p.a, 1, m, p.b, 1, k, p.want, 1, m);
    return p;
}

static void free_problem(Problem* p) {
    free(p->a);
    free(p->b);
    free(p->c);
    free(p->want);
}

static double* block_to_device(const double* g, long ldg, long r0, long rows, long c0, long cols,
                               long ld) {
    double* d = NULL;
    if (cudaMalloc((void**)&d, sizeof(double) * ld * cols) != cudaSuccess) return NULL;
    cudaMemset(d, 0, sizeof(double) * ld * cols);
    cudaMemcpy2D(d, sizeof(double) * ld, g + r0 + c0 * ldg, sizeof(double) * ldg,
                 sizeof(double) * rows, cols, cudaMemcpyHostToDevice);
    return d;
}

/* relative Frobenius error of a device block against the matching block of `want` */
static double block_error(const double* dev, long ld, const double* want, long ldw, long r0,
                          long rows, long c0, long cols) {
    double* h = malloc(sizeof(double) * rows * cols);
    cudaMemcpy2D(h, sizeof(double) * rows, dev, sizeof(double) * ld, sizeof(double) * rows, cols,
                 cudaMemcpyDeviceToHost);
    double err = 0.0;
    strassen_rel_error(rows, cols, h, 1, rows, want + r0 + c0 * ldw, 1, ldw, &err);
    free(h);
    return err;
}

static void run_nccl(strassen_variant variant, int level, long panel) {
    const long m = 384, n = 320, k = 512;
    const double alpha = 0.75;
    Problem p = make_problem(m, n, k, alpha, 11);
    strassen_ctx* ctx = NULL;
    strassen_dist* d = NULL;
    char id[STRASSEN_DIST_ID_BYTES];
    CHECK(strassen_ctx_create(&ctx) == STRASSEN_OK);
    strassen_status st = strassen_dist_unique_id(id);
    if (st != STRASSEN_OK) printf("unique id: %s\n", strassen_last_error());
    CHECK(st == STRASSEN_OK);
    st = strassen_dist_create(&d, ctx, id, 0, 1, 1, 1);
    if (st != STRASSEN_OK) printf("create: %s\n", strassen_last_error());
    CHECK(st == STRASSEN_OK && d != NULL);
    if (d) {
        cudaStream_t s;
        cudaStreamCreate(&s);
        double* da = block_to_device(p.a, m, 0, m, 0, k, m + 2); /* padded lda: the copy path */
        double* db = block_to_device(p.b, k, 0, k, 0, n, k);
        double* dc = block_to_device(p.c, m, 0, m, 0, n, m);
        st = strassen_dist_gemm(d, s, variant, level, m, n, k, alpha, da, m + 2, db, k, dc, m, panel);
        if (st != STRASSEN_OK) printf("dist gemm: %s\n", strassen_last_error());
        CHECK(st == STRASSEN_OK);
        CHECK(cudaStreamSynchronize(s) == cudaSuccess);
        long launches = 0, panels = 0;
        CHECK(strassen_dist_last_counts(d, &launches, &panels) == STRASSEN_OK);
        CHECK(panels == k / (panel ? panel : k) && launches >= panels);
        const double err = block_error(dc, m, p.want, m, 0, m, 0, n);
        printf("nccl 1x1 variant %d level %d panel %ld: rel_err %.3e, %ld launches\n", (int)variant,
               level, panel, err, launches);
        CHECK(err < 1e-11);
        /* validation */
        CHECK(strassen_dist_gemm(d, s, variant, level, m, n, k, alpha, da, m + 2, db, k, dc, m, 7) ==
              STRASSEN_ERR_PARAM);
        CHECK(strassen_dist_gemm(d, s, variant, level, m, n, k, alpha, da, m - 1, db, k, dc, m, 0) ==
              STRASSEN_ERR_PARAM);
        CHECK(strassen_dist_gemm(d, s, variant, level, m, n, k, alpha, p.a, m, db, k, dc, m, 0) ==
              STRASSEN_ERR_PARAM); /* host block */
        CHECK(strassen_dist_gemm(d, s, STRASSEN_DGEMM, 1, m, n, k, alpha, da, m + 2, db, k, dc, m,
                                 0) == STRASSEN_ERR_PARAM);
        cudaFree(da);
        cudaFree(db);
        cudaFree(dc);
        cudaStreamDestroy(s);
    }
    strassen_dist_destroy(d);
    strassen_ctx_destroy(ctx);
    free_problem(&p);
}

static void run_loopback(int pr, int pc, strassen_variant variant, int level, long panel) {
    const long m = 256, n = 384, k = 384;
    const double alpha = -0.5;
    const int P = pr * pc;
    Problem p = make_problem(m, n, k, alpha, 23);
    const long ml = m / pr, nl = n / pc, kc = k / pc, kr = k / pr;
    strassen_ctx* ctx = NULL;
    strassen_dist_mailbox* mb = NULL;
    CHECK(strassen_ctx_create(&ctx) == STRASSEN_OK);
    CHECK(strassen_dist_mailbox_create(&mb) == STRASSEN_OK);
    strassen_dist** d = calloc(P, sizeof *d);
    double **da = calloc(P, sizeof *da), **db = calloc(P, sizeof *db), **dc = calloc(P, sizeof *dc);
    for (int r = 0; r < P; ++r) {
        const int i = r / pc, j = r % pc;
        CHECK(strassen_dist_create_loopback(&d[r], ctx, mb, r, pr, pc) == STRASSEN_OK);
        da[r] = block_to_device(p.a, m, i * ml, ml, j * kc, kc, ml);
        db[r] = block_to_device(p.b, k, i * kr, kr, j * nl, nl, kr + 4); /* padded ldb */
    }
    double worst = 0.0;
    for (int replay = 0; replay < 2; ++replay) {
        CHECK(strassen_dist_mailbox_set_replay(mb, replay) == STRASSEN_OK);
        for (int r = 0; r < P; ++r) {
            const int i = r / pc, j = r % pc;
            if (dc[r]) cudaFree(dc[r]);
            dc[r] = block_to_device(p.c, m, i * ml, ml, j * nl, nl, ml);
            strassen_status st = strassen_dist_gemm(d[r], NULL, variant, level, m, n, k, alpha,
                                                    da[r], ml, db[r], kr + 4, dc[r], ml, panel);
            if (st != STRASSEN_OK) printf("loopback gemm: %s\n", strassen_last_error());
            CHECK(st == STRASSEN_OK);
            CHECK(cudaDeviceSynchronize() == cudaSuccess);
            if (replay) {
                const double err = block_error(dc[r], ml, p.want, m, i * ml, ml, j * nl, nl);
                if (err > worst) worst = err;
            }
        }
    }
    printf("loopback %dx%d variant %d level %d panel %ld: worst block rel_err %.3e\n", pr, pc,
           (int)variant, level, panel, worst);
    CHECK(worst < 1e-11);
    for (int r = 0; r < P; ++r) {
        strassen_dist_destroy(d[r]);
        cudaFree(da[r]);
        cudaFree(db[r]);
        cudaFree(dc[r]);
    }
    free(d);
    free(da);
    free(db);
    free(dc);
    strassen_dist_mailbox_destroy(mb);
    strassen_ctx_destroy(ctx);
    free_problem(&p);
}

int main(int argc, char** argv) {
    const int no_device = argc > 1 && strcmp(argv[1], "--no-device") == 0;
    schedule_checks();
    if (!no_device) {
        run_nccl(STRASSEN_ABC, 2, 128);
        run_nccl(STRASSEN_NAIVE, 1, 0);
        run_loopback(2, 2, STRASSEN_ABC, 1, 96);  /* panels inside one owner */
        run_loopback(2, 4, STRASSEN_AB, 2, 128);  /* panels straddling A owners (k/pc = 96) */
        run_loopback(2, 2, STRASSEN_C, 2, 384);   /* one panel straddling both owners */
        run_loopback(1, 2, STRASSEN_DGEMM, 0, 64);
    }
    printf(failures ? "FAILED (%d)\n" : "PASS\n", failures);
    return failures ? 1 : 0;
}
