/*
 * strassen.h -- C ABI of the B200 (sm_100a) Strassen DGEMM library
 * (libstrassen_b200.so).
 *
 * Drop-in for the reference library's public interface
 * (/root/reference/proj/include/strassen.h, shared target `strassen`,
 * proj/CMakeLists.txt:28-30).  Every declaration in PART 1 keeps the
 * reference's name, argument meaning, status codes and validation order; the
 * comment on each cites the reference declaration (strassen.h:line) and its
 * implementation (capi.cpp:line).  PART 2 adds B200 entry points that the
 * reference does not have (device-pointer / stream entry, column-major dgemm
 * shim with beta, launch accounting).
 *
 * Semantics (reference strassen.h:1-6, matrix.hpp:9-27): all matrices are
 * double precision, addressed as (base pointer, row stride, column stride)
 * in elements; element (i, j) lives at p[i*rs + j*cs]; a transpose is a
 * stride swap.  Every multiply computes C := alpha * A * B + C (no beta).
 *
 * Pointers may be host memory (pageable or pinned) or device memory (cudaMalloc /
 * managed).  Host operands are staged through device memory inside the call;
 * device operands are used in place.  strassen_gemm returns after C is
 * updated (synchronous, like the reference).  There is no CPU fallback: when
 * no CUDA device is usable, compute entry points return STRASSEN_ERR_DEVICE.
 */
#ifndef STRASSEN_B200_H
#define STRASSEN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ============================ PART 1: reference ABI ======================== */

/* reference strassen.h:16-23 */
typedef enum strassen_status {
    STRASSEN_OK = 0,
    STRASSEN_ERR_DIMENSION = 1,
    STRASSEN_ERR_PARAM = 2,
    STRASSEN_ERR_DOMAIN = 3,
    STRASSEN_ERR_ALLOC = 4,
    STRASSEN_ERR_NULL = 5,
    /* B200 addition: CUDA device missing / kernel launch or copy failed. */
    STRASSEN_ERR_DEVICE = 6
} strassen_status;

/* reference strassen.h:25-30 */
typedef enum strassen_variant {
    STRASSEN_DGEMM = 0, /* classical gemm; level must be 0 */
    STRASSEN_ABC = 1,   /* operand sums formed on chip, multi-destination epilogue */
    STRASSEN_AB = 2,    /* operand sums on chip, products to temporaries, streamed C */
    STRASSEN_NAIVE = 3, /* operand sums and products materialised */
    /* B200 addition (not in the reference): operand sums materialised by one
     * batched HBM pass, C updates fused in the epilogue (no product
     * temporaries) -- the fourth point of the paper's fusion design space,
     * and the fastest two-level form on B200. */
    STRASSEN_C = 4
} strassen_variant;

/* reference strassen.h:32-35.  Kept for ABI parity: validated exactly like the
 * reference (all > 0, mc % mr == 0, nc % nr == 0, mr, nr <= 32) and used by
 * the instrumentation counters and the analytical model; the GPU tiling is
 * fixed by the kernels. */
typedef struct strassen_blocking {
    long mc, nc, kc;
    long mr, nr;
} strassen_blocking;

/* reference strassen.h:37-42 */
typedef struct strassen_model_params {
    double tau_a;          /* seconds per flop */
    double tau_b;          /* seconds per 8-byte element from slow memory */
    double lambda;         /* prefetch efficiency on kernel C traffic, [0.5, 1] */
    double channel_factor; /* multiplier on tau_b */
} strassen_model_params;

/* reference strassen.h:44-49 */
typedef struct strassen_breakdown {
    double ta_mul, ta_a_add, ta_b_add, ta_c_add;
    double tm_a_mul, tm_b_mul, tm_c_mul;
    double tm_a_add, tm_b_add, tm_c_add;
    double total;
} strassen_breakdown;

/* reference strassen.h:51-61.  Filled analytically from the operand table and
 * the ctx blocking so the values equal the reference's instrumented counts. */
typedef struct strassen_counter_values {
    int64_t pack_a_calls, pack_b_calls;
    int64_t pack_a_elems, pack_b_elems;
    int64_t pack_a_add_flops, pack_b_add_flops;
    int64_t kernel_calls, kernel_fma_flops;
    int64_t kernel_c_elems, kernel_update_flops;
    int64_t a_plus_passes, a_plus_elems, a_plus_flops;
    int64_t b_plus_passes, b_plus_elems, b_plus_flops;
    int64_t c_plus_passes, c_plus_elems, c_plus_flops;
} strassen_counter_values;

/* Opaque context (reference capi.cpp:12-18): blocking, thread count, counters,
 * plus the B200 state (device workspace, stream, cached plans).  Not safe for
 * concurrent calls (same as the reference). */
typedef struct strassen_ctx strassen_ctx;

strassen_status strassen_ctx_create(strassen_ctx** out);            /* strassen.h:67, capi.cpp:65-69 */
void strassen_ctx_destroy(strassen_ctx* ctx);                      /* strassen.h:68, capi.cpp:71 */
strassen_status strassen_ctx_set_blocking(strassen_ctx* ctx,        /* strassen.h:70-71, capi.cpp:73-81 */
                                          const strassen_blocking* bp);
strassen_status strassen_ctx_get_blocking(const strassen_ctx* ctx,  /* strassen.h:72-73, capi.cpp:83-89 */
                                          strassen_blocking* out);
/* threads >= 1 (capi.cpp:91-96); recorded, the GPU path does not use it. */
strassen_status strassen_ctx_set_threads(strassen_ctx* ctx, int threads);
strassen_status strassen_ctx_enable_counters(strassen_ctx* ctx, int enabled);   /* capi.cpp:98-102 */
strassen_status strassen_ctx_reset_counters(strassen_ctx* ctx);                 /* capi.cpp:104-108 */
strassen_status strassen_ctx_get_counters(const strassen_ctx* ctx,              /* capi.cpp:110-125 */
                                          strassen_counter_values* out);

/* THE HOT PATH.  reference strassen.h:82-86, capi.cpp:127-145.
 * C := alpha A B + C, A m x k, B k x n, C m x n.
 * level: 0 for STRASSEN_DGEMM, 1 or 2 for the Strassen variants.
 * Validation order: NULL ctx/a/b/c -> STRASSEN_ERR_NULL; DGEMM with level != 0
 * or a Strassen variant with level not in {1, 2} -> STRASSEN_ERR_PARAM;
 * m, n or k < 1 -> STRASSEN_ERR_PARAM; invalid ctx blocking -> PARAM;
 * allocation failure -> STRASSEN_ERR_ALLOC; CUDA failure -> STRASSEN_ERR_DEVICE. */
strassen_status strassen_gemm(strassen_ctx* ctx, strassen_variant variant, int level, long m,
                              long n, long k, double alpha, const double* a, long rs_a, long cs_a,
                              const double* b, long rs_b, long cs_b, double* c, long rs_c,
                              long cs_c);

/* Triple-loop oracle on the HOST (strassen.h:89-93, matrix.cpp:37-52):
 * accumulation over p strictly ascending; the rounding reference for tests. */
strassen_status strassen_reference_gemm(long m, long n, long k, double alpha, const double* a,
                                        long rs_a, long cs_a, const double* b, long rs_b,
                                        long cs_b, double* c, long rs_c, long cs_c);

/* ||C_test - C_ref||_F / max(||C_ref||_F, 1) on host buffers
 * (strassen.h:96-99, matrix.cpp:54-66). */
strassen_status strassen_rel_error(long rows, long cols, const double* c_test, long rs_t,
                                   long cs_t, const double* c_ref, long rs_r, long cs_r,
                                   double* out);

/* Analytical model, same coefficients as the reference (strassen.h:102-108,
 * model.cpp:48-134; level 2 uses the paper's 154/462/194). */
strassen_status strassen_model_predict(strassen_variant variant, int level, long m, long n, long k,
                                       const strassen_blocking* bp,
                                       const strassen_model_params* mp,
                                       strassen_breakdown* breakdown_out, double* egf_out);

/* 2mnk / seconds * 1e-9; seconds <= 0 -> STRASSEN_ERR_DOMAIN (model.cpp:113-117). */
strassen_status strassen_effective_gflops(long m, long n, long k, double seconds, double* out);

/* Ivy Bridge single-core preset (strassen.h:112-114, model.cpp:39-46). */
void strassen_model_params_ivy_bridge(strassen_model_params* out);
/* mc=96 nc=4096 kc=256 mr=8 nr=4 (kernel.hpp:11-17). */
void strassen_blocking_defaults(strassen_blocking* out);

/* out = {mults, a_adds, b_adds, c_updates} for level 1 or 2
 * (strassen.h:117-119, table.cpp:104-113): (7,5,5,12) and (49,95,95,144). */
strassen_status strassen_table_counts(int level, long out[4]);

const char* strassen_status_str(strassen_status s);  /* capi.cpp:225-235 */

/* ============================ PART 2: B200 additions ======================= */

/* Device-pointer entry on a caller-provided CUDA stream (cudaStream_t passed
 * as void*, used exactly; NULL = the CUDA legacy default stream).  A, B, C must be device (or managed)
 * memory.  Asynchronous: returns after enqueueing; C is updated in stream
 * order.  Same validation and semantics as strassen_gemm.
 *
 * CUDA graphs: the call may be issued on a stream that is being captured
 * (cudaStreamBeginCapture); its kernels and counter resets become graph nodes and
 * nothing synchronises.  Conditions: the ctx's workspace is already sized (run the
 * same call once before capturing -- a capture that would have to grow it returns
 * STRASSEN_ERR_ALLOC), profiling is off, and whoever replays the graph keeps the
 * replays from overlapping other calls on the same ctx (a captured call cannot wait
 * for, or be waited on by, calls outside its graph).  Replays are bitwise equal to
 * the eager call.  Small problems are bound by host submission (20-60 us per
 * call), which a graph replay removes. */
strassen_status strassen_gemm_device(strassen_ctx* ctx, void* stream, strassen_variant variant,
                                     int level, long m, long n, long k, double alpha,
                                     const double* a, long rs_a, long cs_a, const double* b,
                                     long rs_b, long cs_b, double* c, long rs_c, long cs_c);

/* Column-major BLAS-style shim (the north-star dgemm entry): op(A) = A or A^T
 * per transa ('N'/'n' or 'T'/'t'/'C'/'c'), likewise transb;
 * C := alpha op(A) op(B) + beta C.  beta != 1 pre-scales C on the device
 * (exactly 0 clears it, BLAS convention) before the Strassen call.
 * lda/ldb/ldc >= max(1, rows) else STRASSEN_ERR_PARAM. */
strassen_status strassen_dgemm(strassen_ctx* ctx, strassen_variant variant, int level, char transa,
                               char transb, long m, long n, long k, double alpha, const double* a,
                               long lda, const double* b, long ldb, double beta, double* c,
                               long ldc);

/* Stream used by strassen_gemm / strassen_dgemm (cudaStream_t as void*);
 * default (and NULL) = the CUDA legacy default stream. */
strassen_status strassen_ctx_set_stream(strassen_ctx* ctx, void* stream);

/* Events (cudaEvent_t passed as void*, NULL = none) that the NEXT compute call on
 * this ctx waits on right before its first kernel reading device operand A, B or C:
 * an operand still being produced (a copy or a collective on another stream) then
 * overlaps the work that does not need it -- e.g. C arriving while the operand
 * sums and products run.  Applies to that one call, then cleared. */
strassen_status strassen_ctx_set_operand_events(strassen_ctx* ctx, void* a_ready, void* b_ready,
                                               void* c_ready);

/* Number of CUDA kernels the last compute call on this ctx launched. */
strassen_status strassen_ctx_last_launches(const strassen_ctx* ctx, long* out);

/* Fringe handling for m, n or k not divisible by 2^level: 1 (default) =
 * dynamic peeling (Strassen on the even core + classical fringe updates);
 * 0 = the reference's zero padding of clipped quadrants (matrix.cpp:14-22). */
strassen_status strassen_ctx_set_peeling(strassen_ctx* ctx, int enabled);

/* Host-pointer calls (strassen_gemm / strassen_dgemm with beta == 1) with
 * column-major B and C: 1 (default) = pipeline the call in column windows of
 * the quadrant partition, so B's and C's transfers and C's copy-back overlap
 * the kernels of other windows; 0 = copy everything in, compute, copy out.
 * Results are bitwise identical either way. */
strassen_status strassen_ctx_set_pipelining(strassen_ctx* ctx, int enabled);

/* Highest Strassen level this ctx accepts: 2 (default, the reference's limit,
 * capi.cpp:133-135 / table.cpp:101) or 3.  At 3, STRASSEN_NAIVE and STRASSEN_C
 * also run level 3: one materialised outer level (the one-level table,
 * table.cpp:18-33) over level-2 calls of the same variant, i.e. the 343
 * products of the composed level-3 table (acceptance.cpp:86-88).  ABC / AB at
 * level 3 stay STRASSEN_ERR_PARAM.  Other values: STRASSEN_ERR_PARAM. */
strassen_status strassen_ctx_set_max_level(strassen_ctx* ctx, int max_level);

/* ABC / AB operand sums (the reference's pack_a_sum / pack_b_sum,
 * blocking.cpp:12-66): an operand side of up to max_terms terms is summed in the
 * mm kernel's registers while its term tiles stream in; a longer side is formed
 * by one materialising HBM pass first (materialize_sum, variants.cpp:53-96).
 * Both forms add the terms in listed order with identical roundings, so the
 * result is bitwise the same for every setting; only speed differs.  1..4;
 * default 2 (level 1 fully fused, level 2's 4-term sides materialised:
 * profiles/r02_fuse_probe.log).  Other values: STRASSEN_ERR_PARAM. */
strassen_status strassen_ctx_set_fused_terms(strassen_ctx* ctx, int max_terms);

/* Per-launch CUDA-event timing of the calls on this ctx (off by default).
 * strassen_ctx_last_profile writes a JSON list [{"kernel": name, "ms": t,
 * "start_ms": offset from the first launch}, ...]
 * for the last compute call into buf (NUL-terminated; STRASSEN_ERR_ALLOC if
 * it did not fit).  Synchronises with the recorded events. */
strassen_status strassen_ctx_enable_profiling(strassen_ctx* ctx, int enabled);
strassen_status strassen_ctx_last_profile(strassen_ctx* ctx, char* buf, long size);

/* Device memory currently held by the ctx workspace, in bytes. */
strassen_status strassen_ctx_workspace_bytes(const strassen_ctx* ctx, long* out);

/* Model-guided dispatch (the paper's use of its model,
 * PAPER.md:894-895): the variant and level a B200 cost model, fitted to the
 * measured kernel efficiencies, predicts fastest for an m x n x k multiply,
 * and the predicted seconds (may be NULL).  No device needed. */
/* The B200 cost model's predicted seconds for one configuration on this
 * device (the quantity strassen_select minimises). */
strassen_status strassen_predict_b200(strassen_variant variant, int level, long m, long n, long k,
                                      double* seconds_out);

strassen_status strassen_select(long m, long n, long k, strassen_variant* variant_out,
                                int* level_out, double* seconds_out);

/* strassen_select over the levels this ctx admits (strassen_ctx_set_max_level):
 * with max level 3 the Naive / C level-3 configurations are candidates too.
 * strassen_predict_b200 also accepts level 3 for Naive and C. */
strassen_status strassen_ctx_select(const strassen_ctx* ctx, long m, long n, long k,
                                    strassen_variant* variant_out, int* level_out,
                                    double* seconds_out);

/* Counter values one strassen_gemm(variant, level, m, n, k) call adds under
 * blocking *bp (the analytic instrumentation; no device needed).  Same
 * validation as strassen_gemm for variant / level / dimensions / blocking. */
strassen_status strassen_count_call(strassen_variant variant, int level, long m, long n, long k,
                                    const strassen_blocking* bp, strassen_counter_values* out);

/* Library build string (architecture and kernel configuration). */
const char* strassen_build_info(void);

/* Message of the last failing call on this thread ("" if none). */
const char* strassen_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* STRASSEN_B200_H */
