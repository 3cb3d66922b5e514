// The C ABI (include/strassen.h).  Mirrors the reference's capi.cpp:1-237:
// same validation order and status mapping (guarded(): invalid_argument ->
// PARAM, or DIMENSION when the message says "mismatch"; domain_error ->
// DOMAIN; bad_alloc -> ALLOC), plus STRASSEN_ERR_DEVICE for CUDA failures.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <string_view>
#include <vector>

#include "accounting.hpp"
#include "engine.hpp"
#include "kernels.hpp"
#include "strassen.h"
#include "table.hpp"

struct strassen_ctx {
    strassen_blocking blocking{96, 4096, 256, 8, 4};  // kernel.hpp:11-17
    int threads = 1;
    bool counters_enabled = false;
    strassen_counter_values counters{};
    sb200::Engine engine;
};

static thread_local std::string g_last_error;

namespace sb200 {
void set_last_error(const std::string& what) { g_last_error = what; }  // dist.cpp
}  // namespace sb200

namespace {

template <typename F>
strassen_status guarded(F&& f) {
    try {
        f();
        return STRASSEN_OK;
    } catch (const sb200::Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return std::string_view(e.what()).find("mismatch") != std::string_view::npos
                   ? STRASSEN_ERR_DIMENSION
                   : STRASSEN_ERR_PARAM;
    } catch (const std::domain_error& e) {
        g_last_error = e.what();
        return STRASSEN_ERR_DOMAIN;
    } catch (const std::bad_alloc& e) {
        g_last_error = e.what();
        return STRASSEN_ERR_ALLOC;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return STRASSEN_ERR_PARAM;
    }
}

strassen_status check_variant_level(strassen_variant variant, int level) {
    if (variant == STRASSEN_DGEMM && level != 0) return STRASSEN_ERR_PARAM;
    if (variant != STRASSEN_DGEMM && (level < 1 || level > 2)) return STRASSEN_ERR_PARAM;
    return STRASSEN_OK;
}

void validate_call(strassen_variant variant, long m, long n, long k, const strassen_blocking& bp) {
    if (variant != STRASSEN_DGEMM && variant != STRASSEN_ABC && variant != STRASSEN_AB &&
        variant != STRASSEN_NAIVE && variant != STRASSEN_C)
        throw std::invalid_argument("unknown variant");
    if (m < 1 || n < 1 || k < 1) throw std::invalid_argument("gemm: dimensions must be >= 1");
    sb200::validate_blocking(bp);
    if (m > (1L << 31) - 1 || n > (1L << 31) - 1 || k > (1L << 31) - 1)
        throw std::invalid_argument("gemm: dimensions must be < 2^31");
}

// Element span of a strided view: [lo, hi] offsets from the base pointer.
void span_of(long rows, long cols, long rs, long cs, long& lo, long& hi) {
    lo = hi = 0;
    const long a = (rows - 1) * rs, b = (cols - 1) * cs;
    lo += std::min(0L, a) + std::min(0L, b);
    hi += std::max(0L, a) + std::max(0L, b);
}

// Makes `dev` current for a scope (dev < 0: no change) and restores the caller's device.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        int cur = -1;
        if (dev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != dev &&
            cudaSetDevice(dev) == cudaSuccess)
            prev = cur;
        cudaGetLastError();
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

void cuda_ck(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) throw sb200::Error(STRASSEN_ERR_ALLOC, what);
    if (e != cudaSuccess)
        throw sb200::Error(STRASSEN_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}

// Host operand -> device view (copy of the view's span); device -> as is.
// Host operands are copied on the engine's copy stream (in call order A, B, C)
// and each gets a ready event; kernels wait on it right before their first
// read, so B's and C's transfers overlap the work that does not need them.
sb200::DView stage_in(sb200::Engine& e, cudaStream_t s, const double* p, long rows, long cols,
                      long rs, long cs, sb200::DeviceBuffer& buf, bool copy, bool& staged,
                      cudaEvent_t ready_ev) {
    sb200::DView v;
    v.rows = rows;
    v.cols = cols;
    v.rs = rs;
    v.cs = cs;
    staged = !sb200::is_device_pointer(p);
    if (!staged) {
        v.p = const_cast<double*>(p);
        return v;
    }
    long lo, hi;
    span_of(rows, cols, rs, cs, lo, hi);
    const size_t count = static_cast<size_t>(hi - lo + 1);
    double* d = e.ensure(buf, count * 8);
    (void)s;
    if (copy) {
        cuda_ck(cudaMemcpyAsync(d, p + lo, count * 8, cudaMemcpyHostToDevice, e.copy_stream),
                "H2D operand");
        cuda_ck(cudaEventRecord(ready_ev, e.copy_stream), "ready event");
        v.ready = ready_ev;
    }
    v.p = d - lo;
    return v;
}

strassen_status gemm_impl(strassen_ctx* ctx, bool explicit_stream, cudaStream_t user_stream,
                          bool device_only,
                          strassen_variant variant, int level, long m, long n, long k,
                          double alpha, const double* a, long rs_a, long cs_a, const double* b,
                          long rs_b, long cs_b, double* c, long rs_c, long cs_c, bool has_beta,
                          double beta) {
    if (!ctx || !a || !b || !c) return STRASSEN_ERR_NULL;
    // operand events apply to this call only, whatever its outcome
    const cudaEvent_t ready[3] = {ctx->engine.next_ready[0], ctx->engine.next_ready[1],
                                  ctx->engine.next_ready[2]};
    ctx->engine.next_ready[0] = ctx->engine.next_ready[1] = ctx->engine.next_ready[2] = nullptr;
    if (strassen_status st = check_variant_level(variant, level)) {
        // level 3 (B200 extension) only after strassen_ctx_set_max_level(ctx, 3),
        // and only for the materialising variants (Naive, C)
        const bool l3 = level == 3 && ctx->engine.max_level >= 3 &&
                        (variant == STRASSEN_NAIVE || variant == STRASSEN_C);
        if (!l3) return st;
    }
    return guarded([&] {
        validate_call(variant, m, n, k, ctx->blocking);
        sb200::Engine& e = ctx->engine;
        // a ctx stays on the device it was first used on (its streams, events and
        // buffers live there): run the call there, restore the caller's device after
        const DeviceGuard dev_guard(e.initialised ? e.device : -1);
        e.init();
        cudaStream_t s = explicit_stream ? user_stream : e.stream();
        // device entry: reject host operands before any staging or allocation
        if (device_only && (!sb200::is_device_pointer(a) || !sb200::is_device_pointer(b) ||
                            !sb200::is_device_pointer(c)))
            throw std::invalid_argument("strassen_gemm_device: operands must be device memory");
        // CUDA graph capture (device entry on an explicit stream): the call's launches and
        // counter resets become graph nodes.  Events recorded outside the capture cannot
        // be waited on inside it and vice versa, so a captured call neither waits for the
        // ctx's previous call nor leaves its own completion event; the workspace must
        // already be sized (a warm-up call of the same shape), since growing it
        // synchronises; and whoever replays the graph keeps it from overlapping other
        // work on this ctx (include/strassen.h, strassen_gemm_device).
        bool capturing = false;
        if (s != nullptr) {
            cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
            cuda_ck(cudaStreamIsCapturing(s, &cap), "capture status");
            capturing = cap != cudaStreamCaptureStatusNone;
        }
        e.capturing = capturing;
        if (capturing && (!device_only || e.profiling))
            throw std::invalid_argument(
                "stream capture: only strassen_gemm_device (device operands, no profiling)");
        // the workspace is shared by every call on this ctx: order this call after the
        // previous one even when it was issued on another stream
        if (e.ev_last_recorded && !capturing)
            cuda_ck(cudaStreamWaitEvent(s, e.ev_last, 0), "order after previous call");
        e.unit_ctr_next = 0;
        try {
        long launches = 0;
        bool sa = false, sb = false, sc = false;
        // the copy stream may only overwrite staging buffers once earlier work on s is done
        // (a captured call stages nothing, and an unjoined fork would fail the capture)
        if (!capturing) {
            cuda_ck(cudaEventRecord(e.ev_call, s), "call event");
            cuda_ck(cudaStreamWaitEvent(e.copy_stream, e.ev_call, 0), "copy stream order");
        }
        // Host B and C in column-major layouts: pipeline the call in windows
        // (engine.hpp Windows) when the problem is large enough; A arrives in
        // row strips when it is host column-major too.
        sb200::Windows W;
        const bool a_strips = rs_a == 1 && cs_a >= m && !sb200::is_device_pointer(a);
        if (!device_only && e.pipelining && !(has_beta && beta != 1.0) && rs_b == 1 &&
            rs_c == 1 && cs_b >= k && cs_c >= m && !sb200::is_device_pointer(b) &&
            !sb200::is_device_pointer(c))
            sb200::plan_windows(e, variant, level, m, n, k, a_strips, W);
        const bool windowed = W.count() > 0;
        const bool a_windowed = windowed && W.rows > 1;
        sb200::DView A = stage_in(e, s, a, m, k, rs_a, cs_a, e.stage_a, !a_windowed, sa, e.ev_ready[0]);
        sb200::DView B = stage_in(e, s, b, k, n, rs_b, cs_b, e.stage_b, !windowed, sb, e.ev_ready[1]);
        sb200::DView C = stage_in(e, s, c, m, n, rs_c, cs_c, e.stage_c, !windowed, sc, e.ev_ready[2]);
        // device operands still being produced elsewhere (strassen_ctx_set_operand_events):
        // kernels wait on their event right before first reading them
        if (!sa && ready[0]) A.ready = ready[0];
        if (!sb && ready[1]) B.ready = ready[1];
        if (!sc && ready[2]) C.ready = ready[2];
        for (auto& t : e.timed) {
            cudaEventDestroy(t.start);
            cudaEventDestroy(t.stop);
        }
        e.timed.clear();
        if (windowed) {
            const int L = (variant == STRASSEN_DGEMM) ? 0 : level;
            const long side = 1L << L, qm = (m + side - 1) / side, qn = (n + side - 1) / side;
            // global index ranges of strip w (quadrant bounds b[w], b[w+1]) inside
            // every quadrant block of extent q, clipped to [0, total) and merged
            // when adjacent
            auto ranges = [&](long total, long q, const std::vector<long>& b, int w) {
                std::vector<std::pair<long, long>> out;
                for (long I = 0; I < side; ++I) {
                    const long lo = std::min(total, I * q + b[w]);
                    const long hi = std::min(total, I * q + b[w + 1]);
                    if (lo >= hi) continue;
                    if (!out.empty() && out.back().second == lo) out.back().second = hi;
                    else out.emplace_back(lo, hi);
                }
                return out;
            };
            // rows [i0, i1) x columns [j0, j1) of a column-major view (ld) as one 2-D copy
            auto copy_block = [&](double* dst, const double* src, long ld, long i0, long i1,
                                  long j0, long j1, cudaMemcpyKind kind, cudaStream_t st) {
                const size_t off = static_cast<size_t>(i0 + j0 * ld);
                cuda_ck(cudaMemcpy2DAsync(dst + off, ld * 8, src + off, ld * 8, (i1 - i0) * 8,
                                          j1 - j0, kind, st),
                        kind == cudaMemcpyHostToDevice ? "H2D window" : "D2H window");
            };
            W.a_ready = e.ev_win_a;
            W.b_ready = e.ev_win_b;
            W.c_ready = e.ev_win_c;
            W.done = e.ev_win_done;
            W.issue_a = [&](int r) {
                if (a_windowed)
                    for (auto [i0, i1] : ranges(m, qm, W.rb, r))
                        copy_block(A.p, a, cs_a, i0, i1, 0, k, cudaMemcpyHostToDevice,
                                   e.copy_stream);
                // otherwise A was staged whole (or is resident): the event follows it,
                // and a resident A still being produced (operand event) too
                else if (A.ready)
                    cuda_ck(cudaStreamWaitEvent(e.copy_stream, A.ready, 0), "operand event");
                cuda_ck(cudaEventRecord(e.ev_win_a[r], e.copy_stream), "window event");
            };
            W.issue_b = [&](int cw) {
                for (auto [j0, j1] : ranges(n, qn, W.cb, cw))
                    copy_block(B.p, b, cs_b, 0, k, j0, j1, cudaMemcpyHostToDevice, e.copy_stream);
                cuda_ck(cudaEventRecord(e.ev_win_b[cw], e.copy_stream), "window event");
            };
            auto c_blocks = [&](int w, cudaMemcpyKind kind, cudaStream_t st) {
                const auto rr = ranges(m, qm, W.rb, w / W.cols);
                const auto cc = ranges(n, qn, W.cb, w % W.cols);
                for (auto [i0, i1] : rr)
                    for (auto [j0, j1] : cc)
                        if (kind == cudaMemcpyHostToDevice)
                            copy_block(C.p, c, cs_c, i0, i1, j0, j1, kind, st);
                        else
                            copy_block(c, C.p, cs_c, i0, i1, j0, j1, kind, st);
            };
            W.issue_c = [&](int w) {
                c_blocks(w, cudaMemcpyHostToDevice, e.copy_stream);
                cuda_ck(cudaEventRecord(e.ev_win_c[w], e.copy_stream), "window event");
            };
            W.issue_out = [&](int w) {
                cuda_ck(cudaStreamWaitEvent(e.d2h_stream, e.ev_win_done[w], 0), "window wait");
                c_blocks(w, cudaMemcpyDeviceToHost, e.d2h_stream);
            };
            launches += sb200::run_device(e, s, variant, level, alpha, A, B, C, &W);
            cuda_ck(cudaEventRecord(e.ev_d2h, e.d2h_stream), "d2h event");
            cuda_ck(cudaStreamWaitEvent(s, e.ev_d2h, 0), "d2h wait");
        } else {
            if (has_beta && beta != 1.0) launches += sb200::scale_device(e, s, C, beta);
            launches += sb200::run_device(e, s, variant, level, alpha, A, B, C);
            if (sc) {
                long lo, hi;
                span_of(m, n, rs_c, cs_c, lo, hi);
                sb200::wait_ready(s, C);  // even if no kernel touched C
                cuda_ck(cudaMemcpyAsync(c + lo, C.p + lo, static_cast<size_t>(hi - lo + 1) * 8,
                                        cudaMemcpyDeviceToHost, s),
                        "D2H result");
            }
        }
        if (!capturing) {
            cuda_ck(cudaEventRecord(e.ev_last, s), "call done event");
            e.ev_last_recorded = true;
        }
        if (!device_only) cuda_ck(cudaStreamSynchronize(s), "kernel execution");
        else cuda_ck(cudaGetLastError(), "kernel launch");
        e.last_launches = launches;
        if (ctx->counters_enabled) {
            strassen_counter_values d{};
            sb200::count_call(variant, level, m, n, k, ctx->blocking, d);
            sb200::add_counters(ctx->counters, d);
        }
        } catch (...) {
            // nothing enqueued by this call may outlive it: copies from / to the
            // caller's buffers and kernels reading the workspace (best effort)
            // (a failed capture is the caller's to end: nothing has run)
            if (!capturing) {
                for (cudaStream_t st : {s, e.copy_stream, e.d2h_stream, e.aux_stream})
                    if (st || st == s) cudaStreamSynchronize(st);
                cudaGetLastError();
                if (cudaEventRecord(e.ev_last, s) == cudaSuccess) e.ev_last_recorded = true;
            }
            cudaGetLastError();
            throw;
        }
    });
}

}  // namespace

extern "C" {

strassen_status strassen_ctx_create(strassen_ctx** out) {
    if (!out) return STRASSEN_ERR_NULL;
    *out = new (std::nothrow) strassen_ctx();
    if (!*out) return STRASSEN_ERR_ALLOC;
    if (const char* v = std::getenv("STRASSEN_B200_FUSE_MAX"))  // 1-4 (experiments)
        (*out)->engine.fuse_max_terms = std::max(1, std::min(4, std::atoi(v)));
    return STRASSEN_OK;
}

void strassen_ctx_destroy(strassen_ctx* ctx) { delete ctx; }

strassen_status strassen_ctx_set_blocking(strassen_ctx* ctx, const strassen_blocking* bp) {
    if (!ctx || !bp) return STRASSEN_ERR_NULL;
    return guarded([&] {
        sb200::validate_blocking(*bp);
        ctx->blocking = *bp;
    });
}

strassen_status strassen_ctx_get_blocking(const strassen_ctx* ctx, strassen_blocking* out) {
    if (!ctx || !out) return STRASSEN_ERR_NULL;
    *out = ctx->blocking;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_set_threads(strassen_ctx* ctx, int threads) {
    if (!ctx) return STRASSEN_ERR_NULL;
    if (threads < 1) return STRASSEN_ERR_PARAM;
    ctx->threads = threads;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_enable_counters(strassen_ctx* ctx, int enabled) {
    if (!ctx) return STRASSEN_ERR_NULL;
    ctx->counters_enabled = enabled != 0;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_reset_counters(strassen_ctx* ctx) {
    if (!ctx) return STRASSEN_ERR_NULL;
    ctx->counters = strassen_counter_values{};
    return STRASSEN_OK;
}

strassen_status strassen_ctx_get_counters(const strassen_ctx* ctx, strassen_counter_values* out) {
    if (!ctx || !out) return STRASSEN_ERR_NULL;
    *out = ctx->counters;
    return STRASSEN_OK;
}

strassen_status strassen_gemm(strassen_ctx* ctx, strassen_variant variant, int level, long m,
                              long n, long k, double alpha, const double* a, long rs_a, long cs_a,
                              const double* b, long rs_b, long cs_b, double* c, long rs_c,
                              long cs_c) {
    return gemm_impl(ctx, false, nullptr, false, variant, level, m, n, k, alpha, a, rs_a, cs_a, b,
                     rs_b, cs_b, c, rs_c, cs_c, false, 1.0);
}

strassen_status strassen_gemm_device(strassen_ctx* ctx, void* stream, strassen_variant variant,
                                     int level, long m, long n, long k, double alpha,
                                     const double* a, long rs_a, long cs_a, const double* b,
                                     long rs_b, long cs_b, double* c, long rs_c, long cs_c) {
    return gemm_impl(ctx, true, static_cast<cudaStream_t>(stream), true, variant, level, m, n, k,
                     alpha, a, rs_a, cs_a, b, rs_b, cs_b, c, rs_c, cs_c, false, 1.0);
}

strassen_status strassen_dgemm(strassen_ctx* ctx, strassen_variant variant, int level, char transa,
                               char transb, long m, long n, long k, double alpha, const double* a,
                               long lda, const double* b, long ldb, double beta, double* c,
                               long ldc) {
    if (!ctx || !a || !b || !c) return STRASSEN_ERR_NULL;
    auto trans = [](char t, bool& out) {
        if (t == 'N' || t == 'n') return out = false, true;
        if (t == 'T' || t == 't' || t == 'C' || t == 'c') return out = true, true;
        return false;
    };
    bool ta = false, tb = false;
    if (!trans(transa, ta) || !trans(transb, tb)) return STRASSEN_ERR_PARAM;
    const long arows = ta ? k : m, brows = tb ? n : k;
    if (lda < std::max(1L, arows) || ldb < std::max(1L, brows) || ldc < std::max(1L, m))
        return STRASSEN_ERR_PARAM;
    // column-major storage: element (r, c) of the stored matrix at p[r + c*ld];
    // a transpose is the stride swap (reference strassen.h:1-6).
    const long rs_a = ta ? lda : 1, cs_a = ta ? 1 : lda;
    const long rs_b = tb ? ldb : 1, cs_b = tb ? 1 : ldb;
    return gemm_impl(ctx, false, nullptr, false, variant, level, m, n, k, alpha, a, rs_a, cs_a, b,
                     rs_b, cs_b, c, 1, ldc, true, beta);
}

strassen_status strassen_ctx_set_operand_events(strassen_ctx* ctx, void* a_ready, void* b_ready,
                                               void* c_ready) {
    if (!ctx) return STRASSEN_ERR_NULL;
    ctx->engine.next_ready[0] = static_cast<cudaEvent_t>(a_ready);
    ctx->engine.next_ready[1] = static_cast<cudaEvent_t>(b_ready);
    ctx->engine.next_ready[2] = static_cast<cudaEvent_t>(c_ready);
    return STRASSEN_OK;
}

strassen_status strassen_ctx_set_stream(strassen_ctx* ctx, void* stream) {
    if (!ctx) return STRASSEN_ERR_NULL;
    ctx->engine.user_stream = static_cast<cudaStream_t>(stream);
    ctx->engine.has_user_stream = stream != nullptr;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_last_launches(const strassen_ctx* ctx, long* out) {
    if (!ctx || !out) return STRASSEN_ERR_NULL;
    *out = ctx->engine.last_launches;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_set_peeling(strassen_ctx* ctx, int enabled) {
    if (!ctx) return STRASSEN_ERR_NULL;
    ctx->engine.peeling = enabled != 0;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_set_pipelining(strassen_ctx* ctx, int enabled) {
    if (!ctx) return STRASSEN_ERR_NULL;
    ctx->engine.pipelining = enabled != 0;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_set_max_level(strassen_ctx* ctx, int max_level) {
    if (!ctx) return STRASSEN_ERR_NULL;
    if (max_level < 2 || max_level > 3) return STRASSEN_ERR_PARAM;
    ctx->engine.max_level = max_level;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_set_fused_terms(strassen_ctx* ctx, int max_terms) {
    if (!ctx) return STRASSEN_ERR_NULL;
    if (max_terms < 1 || max_terms > 4) return STRASSEN_ERR_PARAM;
    ctx->engine.fuse_max_terms = max_terms;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_enable_profiling(strassen_ctx* ctx, int enabled) {
    if (!ctx) return STRASSEN_ERR_NULL;
    ctx->engine.profiling = enabled != 0;
    return STRASSEN_OK;
}

strassen_status strassen_ctx_last_profile(strassen_ctx* ctx, char* buf, long size) {
    if (!ctx || !buf) return STRASSEN_ERR_NULL;
    if (size < 1) return STRASSEN_ERR_PARAM;
    const std::string j = ctx->engine.last_profile();
    std::strncpy(buf, j.c_str(), static_cast<size_t>(size - 1));
    buf[size - 1] = 0;
    return static_cast<long>(j.size()) < size ? STRASSEN_OK : STRASSEN_ERR_ALLOC;
}

strassen_status strassen_ctx_workspace_bytes(const strassen_ctx* ctx, long* out) {
    if (!ctx || !out) return STRASSEN_ERR_NULL;
    *out = static_cast<long>(ctx->engine.workspace_bytes());
    return STRASSEN_OK;
}

strassen_status strassen_reference_gemm(long m, long n, long k, double alpha, const double* a,
                                        long rs_a, long cs_a, const double* b, long rs_b,
                                        long cs_b, double* c, long rs_c, long cs_c) {
    if (!a || !b || !c) return STRASSEN_ERR_NULL;
    return guarded([&] {
        if (m < 1 || n < 1 || k < 1) throw std::invalid_argument("gemm: dimensions must be >= 1");
        // matrix.cpp:37-52: per row, accumulate over p ascending into a row buffer
        std::vector<double> acc(static_cast<size_t>(n));
        for (long i = 0; i < m; ++i) {
            std::fill(acc.begin(), acc.end(), 0.0);
            for (long p = 0; p < k; ++p) {
                const double av = a[i * rs_a + p * cs_a];
                for (long j = 0; j < n; ++j) acc[j] += av * b[p * rs_b + j * cs_b];
            }
            for (long j = 0; j < n; ++j) c[i * rs_c + j * cs_c] += alpha * acc[j];
        }
    });
}

strassen_status strassen_rel_error(long rows, long cols, const double* c_test, long rs_t,
                                   long cs_t, const double* c_ref, long rs_r, long cs_r,
                                   double* out) {
    if (!c_test || !c_ref || !out) return STRASSEN_ERR_NULL;
    return guarded([&] {
        double diff2 = 0.0, ref2 = 0.0;
        for (long i = 0; i < rows; ++i)
            for (long j = 0; j < cols; ++j) {
                const double r = c_ref[i * rs_r + j * cs_r];
                const double d = c_test[i * rs_t + j * cs_t] - r;
                diff2 += d * d;
                ref2 += r * r;
            }
        *out = std::sqrt(diff2) / std::max(std::sqrt(ref2), 1.0);
    });
}

strassen_status strassen_model_predict(strassen_variant variant, int level, long m, long n, long k,
                                       const strassen_blocking* bp,
                                       const strassen_model_params* mp,
                                       strassen_breakdown* breakdown_out, double* egf_out) {
    if (!bp || !mp) return STRASSEN_ERR_NULL;
    if (strassen_status st = check_variant_level(variant, level)) return st;
    return guarded([&] {
        if (variant != STRASSEN_DGEMM && variant != STRASSEN_ABC && variant != STRASSEN_AB &&
            variant != STRASSEN_NAIVE)
            throw std::invalid_argument("unknown variant");
        strassen_breakdown bd;
        double egf = 0.0;
        sb200::model_predict(variant, level, m, n, k, *bp, *mp, bd, egf);
        if (breakdown_out) *breakdown_out = bd;
        if (egf_out) *egf_out = egf;
    });
}

strassen_status strassen_effective_gflops(long m, long n, long k, double seconds, double* out) {
    if (!out) return STRASSEN_ERR_NULL;
    return guarded([&] { *out = sb200::effective_gflops(m, n, k, seconds); });
}

void strassen_model_params_ivy_bridge(strassen_model_params* out) {
    if (!out) return;
    *out = {1.0 / 28.32e9, 8.0 / 59.7 * 1e-9, 0.7, 4.0};  // model.cpp:39-46
}

void strassen_blocking_defaults(strassen_blocking* out) {
    if (!out) return;
    *out = {96, 4096, 256, 8, 4};
}

strassen_status strassen_table_counts(int level, long out[4]) {
    if (!out) return STRASSEN_ERR_NULL;
    return guarded([&] {
        const sb200::OpCounts c = sb200::count_ops(sb200::program_for_level(level));
        out[0] = c.mults;
        out[1] = c.a_adds;
        out[2] = c.b_adds;
        out[3] = c.c_updates;
    });
}

const char* strassen_status_str(strassen_status s) {
    switch (s) {
        case STRASSEN_OK: return "ok";
        case STRASSEN_ERR_DIMENSION: return "dimension mismatch";
        case STRASSEN_ERR_PARAM: return "invalid parameter";
        case STRASSEN_ERR_DOMAIN: return "domain error";
        case STRASSEN_ERR_ALLOC: return "allocation failure";
        case STRASSEN_ERR_NULL: return "null argument";
        case STRASSEN_ERR_DEVICE: return "CUDA device error";
    }
    return "unknown";
}

static int device_sms() {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    else
        cudaGetLastError();
    return sms > 0 ? sms : 148;
}

strassen_status strassen_predict_b200(strassen_variant variant, int level, long m, long n, long k,
                                      double* seconds_out) {
    if (!seconds_out) return STRASSEN_ERR_NULL;
    if (strassen_status st = check_variant_level(variant, level))
        if (!(level == 3 && (variant == STRASSEN_NAIVE || variant == STRASSEN_C))) return st;
    if (m < 1 || n < 1 || k < 1) return STRASSEN_ERR_PARAM;
    *seconds_out = sb200::b200_predict_seconds(variant, level, m, n, k, device_sms());
    return STRASSEN_OK;
}

strassen_status strassen_ctx_select(const strassen_ctx* ctx, long m, long n, long k,
                                    strassen_variant* variant_out, int* level_out,
                                    double* seconds_out) {
    if (!ctx || !variant_out || !level_out) return STRASSEN_ERR_NULL;
    if (m < 1 || n < 1 || k < 1) return STRASSEN_ERR_PARAM;
    double t = 0.0;
    sb200::b200_select(m, n, k, device_sms(), *variant_out, *level_out, t,
                       ctx->engine.max_level);
    if (seconds_out) *seconds_out = t;
    return STRASSEN_OK;
}

strassen_status strassen_select(long m, long n, long k, strassen_variant* variant_out,
                                int* level_out, double* seconds_out) {
    if (!variant_out || !level_out) return STRASSEN_ERR_NULL;
    if (m < 1 || n < 1 || k < 1) return STRASSEN_ERR_PARAM;
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    else
        cudaGetLastError();
    double t = 0.0;
    sb200::b200_select(m, n, k, sms > 0 ? sms : 148, *variant_out, *level_out, t);
    if (seconds_out) *seconds_out = t;
    return STRASSEN_OK;
}

strassen_status strassen_count_call(strassen_variant variant, int level, long m, long n, long k,
                                    const strassen_blocking* bp, strassen_counter_values* out) {
    if (!bp || !out) return STRASSEN_ERR_NULL;
    if (strassen_status st = check_variant_level(variant, level))  // level 3: Naive / C
        if (!(level == 3 && (variant == STRASSEN_NAIVE || variant == STRASSEN_C))) return st;
    return guarded([&] {
        validate_call(variant, m, n, k, *bp);
        strassen_counter_values d{};
        sb200::count_call(variant, level, m, n, k, *bp, d);
        *out = d;
    });
}

const char* strassen_build_info(void) {
    static const std::string info = [] {
        return std::string("libstrassen_b200 sm_100a; mm_kernel tile ") + std::to_string(sb200::kBM) +
               "x" + std::to_string(sb200::kBN) + "x" + std::to_string(sb200::kBK) +
               " DMMA.8 (mma.sync m8n8k4 f64); TMA ring " + std::to_string(sb200::kRawSlots) +
               " x 16 KB of operand-term tiles; operand sums formed in registers by the " +
               std::to_string(sb200::kConsumerWarps) + " DMMA warps; 1 TMA warp";
    }();
    return info.c_str();
}

const char* strassen_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
