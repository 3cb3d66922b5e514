// Host engine (see engine.hpp).
#include "engine.hpp"

#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <cstdio>
#include <cstdlib>

#include "kernels.hpp"
#include "plan.hpp"
#include "table.hpp"

namespace sb200 {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) throw Error(STRASSEN_ERR_ALLOC, what);
    if (e != cudaSuccess)
        throw Error(STRASSEN_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) throw Error(STRASSEN_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// Column-major (rows x cols, leading dimension ld) fp64 tensor map.
// swizzle_bytes: 128 (boxes of 128-byte rows), 64 (B half tiles) or 0.
void encode_map(CUtensorMap* map, const double* base, long rows, long cols, long long ld,
                uint32_t box0, uint32_t box1, int swizzle_bytes) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                             const_cast<double*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE,
                             swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                             : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                   : CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(STRASSEN_ERR_DEVICE, "cuTensorMapEncodeTiled failed");
}

long ceil_div(long a, long b) { return (a + b - 1) / b; }
long clip(long v, long lo, long hi) { return std::max(lo, std::min(hi, v)); }

// An operand prepared for TMA: column-major, 16-byte aligned quadrant origins.
struct TmaOperand {
    const double* base = nullptr;
    cudaEvent_t ready = nullptr;  // pending copy-in of the operand (read in place)
    long long ld = 0;
    long q_rows_al = 0;  // row offset between quadrant rows (>= logical q rows)
    long rows = 0, cols = 0;
    long q_rows = 0, q_cols = 0;  // logical quadrant extents
};

bool tma_ready(const DView& v, long q_rows, int side) {
    const uintptr_t addr = reinterpret_cast<uintptr_t>(v.p);
    if (v.rs != 1) return false;
    if (v.cs < v.rows || (v.cs % 2) != 0) return false;
    if (addr % 16 != 0) return false;
    if (side > 1 && (q_rows % 2) != 0) return false;
    if (v.cs * 8 >= (1LL << 40)) return false;
    return true;
}

TmaOperand prepare(Engine& e, cudaStream_t s, const DView& v, long q_rows, long q_cols, int side,
                   DeviceBuffer& scratch, long& launches) {
    TmaOperand t;
    t.rows = v.rows;
    t.cols = v.cols;
    t.q_rows = q_rows;
    t.q_cols = q_cols;
    if (tma_ready(v, q_rows, side)) {
        t.ready = v.ready;
        t.base = v.p;
        t.ld = v.cs;
        t.q_rows_al = q_rows;
        return t;
    }
    // Normalise into column-major with each quadrant row block at a 32-byte
    // aligned offset: O(rows*cols) copy, negligible against the O(mnk) work.
    const long q_al = (side > 1) ? ((q_rows + 3) / 4) * 4 : q_rows;
    long long ld = static_cast<long long>(side > 1 ? q_al * side : v.rows);
    ld = std::max<long long>(((ld + 3) / 4) * 4, 4);
    double* dst = e.ensure(scratch, static_cast<size_t>(ld) * v.cols * 8);
    wait_ready(s, v);
    e.prof_begin("repack_kernel", s);
    ck(launch_repack(v.p, v.rs, v.cs, v.rows, v.cols, dst, ld, side > 1 ? q_rows : v.rows + 1,
                     side > 1 ? q_al : v.rows + 1, s),
       "repack");
    e.prof_end(s);
    ++launches;
    t.base = dst;
    t.ld = ld;
    t.q_rows_al = q_al;
    return t;
}

// Quadrant (I, J) of a prepared operand: origin and clipped extent.
const double* quad_origin(const TmaOperand& t, long I, long J) {
    return t.base + I * t.q_rows_al + J * t.q_cols * t.ld;
}
long quad_rows(const TmaOperand& t, long I) { return clip(t.rows - I * t.q_rows, 0, t.q_rows); }
long quad_cols(const TmaOperand& t, long J) { return clip(t.cols - J * t.q_cols, 0, t.q_cols); }

struct QuadView {
    double* p;
    long rows, cols;
};

QuadView c_quad(const DView& C, long qm, long qn, long I, long J) {
    QuadView q;
    q.rows = clip(C.rows - I * qm, 0, qm);
    q.cols = clip(C.cols - J * qn, 0, qn);
    q.p = (q.rows > 0 && q.cols > 0) ? C.p + I * qm * C.rs + J * qn * C.cs : C.p;
    return q;
}

const Program& program(int level) {
    static const Program p0 = identity_program();
    return level == 0 ? p0 : program_for_level(level);
}

// Filter one product's terms to the non-empty quadrants (reference
// all_empty / clamped packing, variants.cpp:26-47, blocking.cpp:21-22: an
// empty view contributes exactly nothing).
Terms live_terms(const Terms& t, const std::vector<bool>& nonempty) {
    Terms out;
    for (const auto& x : t)
        if (nonempty[x.first]) out.push_back(x);
    return out;
}

void fill_desc(ProductDesc& d, const Terms& a, const Terms& b, const Terms& c) {
    std::memset(&d, 0, sizeof(d));
    d.na = static_cast<int8_t>(a.size());
    d.nb = static_cast<int8_t>(b.size());
    d.nc = static_cast<int8_t>(c.size());
    // 4 + 4 terms: stream 8-k half tiles (kernels.cu product_kloop_half; measured
    // slower for 4 + 2, whose 16-k steps already leave the ring 8 slots ahead)
    d.half = (a.size() == 4 && b.size() == 4) ? 1 : 0;
    for (size_t u = 0; u < a.size(); ++u) {
        d.aq[u] = static_cast<int8_t>(a[u].first);
        d.as[u] = static_cast<int8_t>(a[u].second);
    }
    for (size_t u = 0; u < b.size(); ++u) {
        d.bq[u] = static_cast<int8_t>(b[u].first);
        d.bs[u] = static_cast<int8_t>(b[u].second);
    }
    for (size_t u = 0; u < c.size(); ++u) {
        d.cq[u] = static_cast<int8_t>(c[u].first);
        d.cs[u] = static_cast<int8_t>(c[u].second);
    }
}

}  // namespace

// ------------------------------------------------------------------ Engine --
Engine::~Engine() {
    if (!initialised) return;
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (ev_call) cudaEventDestroy(ev_call);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    for (auto ev : ev_ready)
        if (ev) cudaEventDestroy(ev);
    if (aux_stream) cudaStreamDestroy(aux_stream);
    for (cudaEvent_t* arr : {ev_win_a, ev_win_b, ev_sum_a, ev_sum_b})
        for (int w = 0; w < kMaxStrips; ++w)
            if (arr[w]) cudaEventDestroy(arr[w]);
    for (cudaEvent_t* arr : {ev_win_c, ev_win_done})
        for (int w = 0; w < kMaxWindows; ++w)
            if (arr[w]) cudaEventDestroy(arr[w]);
    for (cudaEvent_t ev : {ev_d2h, ev_fork, ev_join})
        if (ev) cudaEventDestroy(ev);
    if (ev_last) cudaEventDestroy(ev_last);
    for (DeviceBuffer* b : {&stage_a, &stage_b, &stage_c, &pack_a, &pack_b, &mbuf, &tabuf, &tbbuf, &ticket_buf,
                               &pack_a3, &pack_b3, &l3_a, &l3_b, &l3_m, &unit_ctr_buf, &fringe_buf})
        if (b->ptr) cudaFree(b->ptr);
}

void Engine::init() {
    if (initialised) return;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw Error(STRASSEN_ERR_DEVICE, "no CUDA device");
    ck(cudaGetDevice(&device), "cudaGetDevice");
    ck(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device), "SM count");
    ck(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking), "copy stream");
    ck(cudaEventCreateWithFlags(&ev_call, cudaEventDisableTiming), "event");
    for (auto& ev : ev_ready) ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    ck(cudaStreamCreateWithFlags(&d2h_stream, cudaStreamNonBlocking), "d2h stream");
    ck(cudaStreamCreateWithFlags(&aux_stream, cudaStreamNonBlocking), "aux stream");
    for (cudaEvent_t* ev : {&ev_d2h, &ev_fork, &ev_join, &ev_last})
        ck(cudaEventCreateWithFlags(ev, cudaEventDisableTiming), "event");
    for (cudaEvent_t* arr : {ev_win_a, ev_win_b, ev_sum_a, ev_sum_b})
        for (int w = 0; w < kMaxStrips; ++w)
            ck(cudaEventCreateWithFlags(&arr[w], cudaEventDisableTiming), "event");
    for (cudaEvent_t* arr : {ev_win_c, ev_win_done})
        for (int w = 0; w < kMaxWindows; ++w)
            ck(cudaEventCreateWithFlags(&arr[w], cudaEventDisableTiming), "event");
    initialised = true;
}

void Engine::prof_begin(const char* name, cudaStream_t s) {
    if (!profiling) return;
    Timed t{name, nullptr, nullptr};
    cudaEventCreate(&t.start);
    cudaEventCreate(&t.stop);
    cudaEventRecord(t.start, s);
    timed.push_back(t);
}

void Engine::prof_end(cudaStream_t s) {
    if (!profiling || timed.empty()) return;
    cudaEventRecord(timed.back().stop, s);
}

std::string Engine::last_profile() {
    std::string out = "[";
    for (size_t i = 0; i < timed.size(); ++i) {
        float ms = -1.0f;
        if (cudaEventSynchronize(timed[i].stop) == cudaSuccess)
            cudaEventElapsedTime(&ms, timed[i].start, timed[i].stop);
        float at = 0.0f;  // start relative to the call's first timed launch
        if (i > 0) cudaEventElapsedTime(&at, timed[0].start, timed[i].start);
        out += (i ? ", " : "") + std::string("{\"kernel\": \"") + timed[i].name +
               "\", \"ms\": " + std::to_string(ms) + ", \"start_ms\": " + std::to_string(at) +
               "}";
    }
    return out + "]";
}

// The synchronous entry points run on the ctx stream: the one set with
// strassen_ctx_set_stream, else the CUDA legacy default stream (which orders
// against the caller's work on other blocking streams).
cudaStream_t Engine::stream() { return has_user_stream ? user_stream : nullptr; }

double* Engine::ensure(DeviceBuffer& b, size_t bytes) {
    if (bytes == 0) bytes = 8;
    if (b.bytes < bytes) {
        if (capturing)
            throw Error(STRASSEN_ERR_ALLOC,
                        "stream capture: the workspace must already be sized (run the same "
                        "call once before capturing it)");
        if (b.ptr) {
            // earlier launches (on any stream) may still read it
            ck(cudaDeviceSynchronize(), "sync before realloc");
            cudaFree(b.ptr);
            b.ptr = nullptr;
            b.bytes = 0;
        }
        const cudaError_t err = cudaMalloc(&b.ptr, bytes);
        if (err != cudaSuccess) {
            b.ptr = nullptr;
            cudaGetLastError();
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            throw Error(err == cudaErrorMemoryAllocation ? STRASSEN_ERR_ALLOC : STRASSEN_ERR_DEVICE,
                        "cudaMalloc workspace: " + std::to_string(bytes >> 20) + " MiB requested, " +
                            std::to_string(fr >> 20) + " MiB free");
        }
        b.bytes = bytes;
    }
    return static_cast<double*>(b.ptr);
}

size_t Engine::workspace_bytes() const {
    size_t t = 0;
    for (const DeviceBuffer* b : {&stage_a, &stage_b, &stage_c, &pack_a, &pack_b, &mbuf, &tabuf, &tbbuf, &ticket_buf,
                               &pack_a3, &pack_b3, &l3_a, &l3_b, &l3_m, &unit_ctr_buf, &fringe_buf})
        t += b->bytes;
    return t;
}

bool is_device_pointer(const void* p) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// SB200_TRACE builds: the device buffer the next mm launch records CTA events into
// (STRASSEN_B200_TRACE_PTR, an address set by tools/cta_trace.py; read per launch)
unsigned long long* trace_buffer() {
#ifdef SB200_TRACE
    if (const char* v = std::getenv("STRASSEN_B200_TRACE_PTR"))
        return reinterpret_cast<unsigned long long*>(std::strtoull(v, nullptr, 0));
#endif
    return nullptr;
}

// A zeroed unit counter for a persistent mm launch on s (MMParams::unit_counter):
// distinct per launch within a call (windows run on two streams), reused across
// calls, which are ordered after each other (gemm_impl's ev_last).
int* next_unit_counter(Engine& e, cudaStream_t s) {
    static const bool dyn_on = [] {
        const char* v = std::getenv("STRASSEN_B200_DYN");  // 0 / 1 (experiments)
        return v ? std::atoi(v) != 0 : true;
    }();
    if (!dyn_on) return nullptr;  // fixed unit stride
    constexpr int kCounters = 1024;
    int* base = reinterpret_cast<int*>(e.ensure(e.unit_ctr_buf, kCounters * sizeof(int)));
    int* c = base + (e.unit_ctr_next++ % kCounters);
    ck(cudaMemsetAsync(c, 0, sizeof(int), s), "unit counter reset");
    return c;
}

// Launch plan of P (ABC / DGEMM / C / AB / Naive), decided on the WHOLE problem
// so that a column window computes exactly what the unwindowed call does:
// tile ownership with the multi-destination epilogue, or -- when the output has
// fewer than two waves of tiles, or the variant stores products (AB, Naive) --
// split mode: one CTA per (tile, product, k-chunk) into partials M_{p,s}, then
// one deterministic stream pass (partials summed in s order, destinations
// applied in table order).
struct FusedPlan {
    bool split = false;
    bool streamk = false;    // split mode: stream-K pieces (kernels.cu)
    bool sk_store = false;   // stream-K of a store-mode program: M_p fixed up in-kernel
    long long part_off = 0;  // partial slots' offset from M (sk_store)
    int sk_len = 0, sk_maxp = 0, sk_grid = 0;
    bool fixup = false;      // split mode finished in the epilogue (no stream pass)
    int* arrive = nullptr;   // per (tile, product) chunk-arrival counters
    int* tickets = nullptr;  // ordered product-parallel fused epilogue (see kernels.hpp)
    int ticket_ld = 0;
    int ksplit = 1, per = 0;
    long long ldm = 0, mstride = 0;
    double* M = nullptr;
    // classical hybrid (plan.hpp choose_tail): the fused tile-owner grid on the tile
    // columns before tail_tn0, stream-K pieces (sk_*, ksplit, M, arrive above) on the rest
    bool tail = false;
    int tail_tn0 = 0;
};

// nprod_plan / terms_plan: plan as for this many products with this mean term
// count (a product group of a larger program plans like the whole program, so
// its k-chunks -- and results -- are the same); 0 = P's own.
FusedPlan plan_fused(Engine& e, cudaStream_t s, const MMParams& P, bool force_split,
                     int nprod_plan = 0, double terms_plan = 0.0, bool windowed = false) {
    FusedPlan F;
    const int ntiles = P.tiles_m * P.tiles_n;
    // (narrow tiles: two resident CTAs per SM)
    const int sms = (e.num_sms > 0 ? e.num_sms : 148) * (P.narrow ? 2 : 1);
    double terms = 0.0;  // mean operand terms per side: fused sums lengthen a k-tile
    for (int p = 0; p < P.nprod; ++p) terms += 0.5 * (P.prod[p].na + P.prod[p].nb);
    terms /= P.nprod > 0 ? P.nprod : 1;
    if (terms_plan > 0.0) terms = terms_plan;
    const int np = nprod_plan > 0 ? nprod_plan : P.nprod;
    long per = P.ktiles;
    const int ks = choose_ksplit(ntiles, np, P.ktiles, sms, static_cast<double>(P.qm) * P.qn,
                                 1.0 + 0.15 * (terms - 1.0), &per);
    // Fused epilogue when the output has >= 2 waves of tiles, or -- for a
    // multi-product program -- when the cost model would not split k anyway: the
    // ticketed (tile, product) grid then has the same CTAs as split mode without
    // its partials and stream pass (8192^3 C L2: 12544 CTAs on 256 tiles).
    // (>= one wave of tiles: with fewer, many products of one tile are in flight
    // at once and their ticketed epilogues serialise -- 1024^3 ABC L2 0.14 -> 0.60 ms)
    bool fused = ntiles >= 2 * sms || (np > 1 && ks == 1 && ntiles >= sms);
    static const bool fixup_on = [] {
        const char* v = std::getenv("STRASSEN_B200_FIXUP");  // 0 / 1 (experiments)
        return v ? std::atoi(v) != 0 : true;
    }();
    static const bool streamk_on = [] {
        const char* v = std::getenv("STRASSEN_B200_STREAMK");  // 0 / 1 (experiments)
        return v ? std::atoi(v) != 0 : true;
    }();
    // Classical launches of two to four waves of tiles: tile ownership quantises to whole
    // waves (2304^3 is 324 tiles on 148 SMs: three waves for 2.19 waves of work, 25.5
    // TF/s against cuBLAS's 33.9; profiles/r02_mid_scan.log).  Stream-K over all the tiles
    // instead, where the cost comparison says so.  Under four waves only: from there host
    // calls run in windows (plan_windows), which cannot run the whole call's pieces, and
    // host and device calls must plan alike.
    bool sk_wide = false;
    static const bool sk_wide_on = [] {
        const char* v = std::getenv("STRASSEN_B200_STREAMK_WIDE");  // 0 / 1 (experiments)
        return v ? std::atoi(v) != 0 : true;
    }();
    if (fused && !force_split && np == 1 && P.nprod == 1 && fixup_on && streamk_on && sk_wide_on &&
        !windowed && ntiles < 4 * sms) {
        const long total = static_cast<long>(ntiles) * P.ktiles;
        const long len = ceil_div(total, std::max(1L, std::min<long>(sms, total / 8)));
        const double t_k = 2.1e-6, t_cta = 3e-6;
        const double t_uni = std::ceil(static_cast<double>(ntiles) / sms) *
                             (static_cast<double>(P.ktiles) * t_k + t_cta);
        const double t_sk = static_cast<double>(len) * t_k +
                            std::ceil(static_cast<double>(len) / P.ktiles + 1.0) * t_cta + 15e-6;
        if (t_sk < 0.97 * t_uni) {
            fused = false;
            sk_wide = true;
        }
    }
    if (fused && !force_split && np == 1 && P.nprod == 1 && fixup_on && streamk_on && sk_wide_on &&
        !windowed && !P.narrow && ntiles >= 4 * sms) {
        // Four waves of tiles and more: whole waves of tile owners, then the last tile
        // columns as stream-K pieces (plan.hpp choose_tail; 3840^3: 7 waves of owners ->
        // 6 waves + a balanced tail).  Not for windowed host calls, whose windows cannot
        // run a whole call's pieces: those keep the plain grid, so at these shapes a
        // pipelined host call and the device call round differently (both within bounds).
        const TailPlan T = choose_tail(P.tiles_m, P.tiles_n, P.ktiles, sms);
        if (T.cols > 0) {
            F.tail = true;
            F.tail_tn0 = P.tiles_n - static_cast<int>(T.cols);
            const long tail_tiles = static_cast<long>(P.tiles_m) * T.cols;
            const long total = tail_tiles * P.ktiles;
            const long len = ceil_div(total, std::max(1L, std::min<long>(sms, total / 8)));
            F.sk_len = static_cast<int>(len);
            F.sk_grid = static_cast<int>(ceil_div(total, len));
            F.sk_maxp = static_cast<int>(ceil_div(len, P.ktiles) + 1);
            F.ksplit = static_cast<int>(ceil_div(P.ktiles, len) + 1);  // partial slots per tile
            F.per = P.ktiles;
            F.ldm = (P.qm + 1) / 2 * 2;
            // partial slots span the tail's columns only (the kernel indexes by the
            // quadrant column: run_fused_window shifts the base)
            F.mstride = F.ldm * static_cast<long long>(T.cols) * kBN;
            F.M = e.ensure(e.mbuf, static_cast<size_t>(F.mstride) * F.ksplit * 8);
            const size_t nt = static_cast<size_t>(P.tiles_m) * P.tiles_n;
            F.arrive = reinterpret_cast<int*>(e.ensure(e.ticket_buf, nt * sizeof(int)));
            ck(cudaMemsetAsync(F.arrive, 0, nt * sizeof(int), s), "arrive reset");
            F.ticket_ld = P.tiles_n;
        }
        return F;
    }
    if (fused && !force_split) {
        // Fused epilogue.  Tile ownership (one CTA walks every product of its
        // tile) quantises to whole waves of CTAs that each run all 7^L products
        // (ABC L2 at 9216^3: 2.2 waves -> 3).  One CTA per (tile, product) with
        // the C updates ordered per tile by tickets applies the same updates in
        // the same order -- bitwise the same result -- and measured faster at
        // every size (16384^3 ABC L2 240.0 -> 238.8 ms, 9216^3 59.0 -> 43.9 ms).
        bool ticketed = P.nprod > 1;
        if (const char* m = std::getenv("STRASSEN_B200_RMW"))  // "owner" / "ticket" (experiments)
            ticketed = P.nprod > 1 && std::strcmp(m, "ticket") == 0 ? true
                       : std::strcmp(m, "owner") == 0             ? false
                                                                   : ticketed;
        if (ticketed) {  // one ticket per C tile
            const size_t nt = static_cast<size_t>(P.tiles_m) * P.tiles_n;
            F.ticket_ld = P.tiles_n;
            F.tickets = reinterpret_cast<int*>(e.ensure(e.ticket_buf, nt * sizeof(int)));
            ck(cudaMemsetAsync(F.tickets, 0, nt * sizeof(int), s), "ticket reset");
        }
        return F;
    }
    F.ksplit = ks;
    F.per = static_cast<int>(per);
    F.split = true;
    F.ldm = (P.qm + 1) / 2 * 2;  // even: 16-B stores
    F.mstride = F.ldm * P.qn;
    if (const char* v = std::getenv("STRASSEN_B200_MPAD"))  // doubles (experiments)
        F.mstride += std::atol(v);
    F.M = e.ensure(e.mbuf, static_cast<size_t>(F.mstride) * P.nprod * F.ksplit * 8);
    // Classical (one product): the last k-chunk CTA of each tile sums the
    // partials in chunk order and applies the C update -- the stream pass's
    // arithmetic, in its order, without its launch (1024^3 105 -> 98 us, 2048^3
    // 598 -> 575 us).  Not for Strassen programs: their 7^L updates per tile
    // would serialise on the tile's ticket (1024^3 ABC L2 139 -> 696 us), where
    // the stream pass applies them in parallel over elements.
    if (sk_wide) {  // (decided above: one chunk per tile would be the alternative)
        F.ksplit = 1;
        F.per = P.ktiles;
        F.streamk = true;
    } else if (!force_split && fixup_on && np == 1 && streamk_on) {
        // Stream-K: the flattened (tile, k-step) space cut into equal ranges, one
        // per persistent CTA, so every SM gets the same work (uniform k-chunks
        // quantise to whole waves: 2048^3 has 256 tiles on 148 SMs).  Pieces of a
        // tile are summed in k order by the last to arrive: deterministic.
        const long total = static_cast<long>(ntiles) * P.ktiles;
        const long min_piece = 8;  // k-steps: prologue and partial traffic stay small
        const long want = std::max(1L, std::min<long>(sms, total / min_piece));
        const long len = ceil_div(total, want);
        // worth it only where whole-wave quantisation of the k-chunk plan costs more
        // than the pieces' partial round trip (~15 us): 2048^3 570 -> 518 us, while
        // 1536^3 (144 tiles, one full wave) got slower (219 -> 232 us)
        const double t_k = 2.1e-6, t_cta = 3e-6;
        const double t_uni = std::ceil(static_cast<double>(ntiles) * ks / sms) *
                                 (static_cast<double>(per) * t_k + t_cta) +
                             (ks > 1 ? 15e-6 : 0.0);  // k-chunks take the same partial fixup
        const double t_sk = static_cast<double>(len) * t_k + t_cta + 15e-6;
        if (t_sk < 0.97 * t_uni) F.streamk = true;
    }
    // (under 4 waves of (tile, product) units only: the host pipeline windows AB /
    // Naive calls from 4 waves up, and a window cannot run the whole call's pieces)
    if ((force_split || np > 1) && streamk_on && !windowed && np == P.nprod &&
        static_cast<long>(ntiles) * np < 4L * sms) {
        // Stream-K for store-mode programs (few tiles, products into temporaries,
        // then the stream pass): the flattened (product, tile, k-step) space cut into
        // equal ranges, one per persistent CTA; the last piece of a (tile, product)
        // sums the pieces in k order and stores M_p.  Uniform k-chunks of 7^L x tiles
        // CTAs quantise to whole waves (1024^3 ABC L1: 112 CTAs of 32 k-steps on 148
        // SMs).  Fused sums lengthen a k-step (term_factor as choose_ksplit).
        const long total = static_cast<long>(ntiles) * np * P.ktiles;
        const long want = std::max(1L, std::min<long>(sms, total / 8));
        const long len = ceil_div(total, want);
        const double t_k = 2.1e-6 * (1.0 + 0.15 * (terms - 1.0)), t_cta = 3e-6;
        const double t_uni = std::ceil(static_cast<double>(ntiles) * np * ks / sms) *
                             (static_cast<double>(per) * t_k + t_cta);
        // a CTA's range spans len / K + 1 pieces, each with its prologue and epilogue
        const double t_sk = static_cast<double>(len) * t_k +
                            std::ceil(static_cast<double>(len) / P.ktiles + 1.0) * t_cta +
                            6e-6;  // + the fixup's partial round trip
        if (t_sk < 0.97 * t_uni) {
            F.streamk = F.sk_store = true;
            F.sk_len = static_cast<int>(len);
            F.sk_grid = static_cast<int>(ceil_div(total, len));
            F.sk_maxp = static_cast<int>(ceil_div(len, P.ktiles) + 1);
            F.ksplit = static_cast<int>(ceil_div(P.ktiles, len) + 1);  // partial slots
            F.per = P.ktiles;
            F.part_off = static_cast<long long>(P.nprod) * F.mstride;
            F.M = e.ensure(e.mbuf, static_cast<size_t>(F.mstride) * P.nprod * (1 + F.ksplit) * 8);
            const size_t na = static_cast<size_t>(P.tiles_m) * P.tiles_n * P.nprod;
            F.arrive = reinterpret_cast<int*>(e.ensure(e.ticket_buf, na * sizeof(int)));
            ck(cudaMemsetAsync(F.arrive, 0, na * sizeof(int), s), "arrive reset");
            F.ticket_ld = P.tiles_n;
            return F;
        }
    }
    if (F.streamk) {
        const long total = static_cast<long>(ntiles) * P.ktiles;
        const long len = ceil_div(total, std::max(1L, std::min<long>(sms, total / 8)));
        F.sk_len = static_cast<int>(len);
        F.sk_grid = static_cast<int>(ceil_div(total, len));
        F.sk_maxp = static_cast<int>(ceil_div(len, P.ktiles) + 1);
        F.ksplit = static_cast<int>(ceil_div(P.ktiles, len) + 1);  // partial slots per tile
        F.per = P.ktiles;
        F.M = e.ensure(e.mbuf, static_cast<size_t>(F.mstride) * F.ksplit * 8);
    }
    if (!force_split && fixup_on && np == 1) {
        // per-tile tickets, then per-(tile, product) arrival counters
        const size_t nt = static_cast<size_t>(P.tiles_m) * P.tiles_n;
        const size_t words = nt * (1 + static_cast<size_t>(P.nprod));
        int* buf = reinterpret_cast<int*>(e.ensure(e.ticket_buf, words * sizeof(int)));
        ck(cudaMemsetAsync(buf, 0, words * sizeof(int), s), "ticket reset");
        F.fixup = true;
        F.tickets = buf;
        F.arrive = buf + nt;
        F.ticket_ld = P.tiles_n;
    }
    return F;
}

// The stream pass of a split / store-mode plan: C_q += alpha gamma M_p over the window,
// each quadrant's updates in table order.
void build_stream_params(StreamParams& S, const MMParams& P, const FusedPlan& F,
                         const std::vector<Terms>& dests, const std::vector<QuadView>& cq,
                         const DView& C, double alpha, long r0, long r1, long c0, long c1) {
    std::memset(&S, 0, sizeof(S));
    S.rs_c = C.rs;
    S.cs_c = C.cs;
    S.alpha = alpha;
    S.ldm = F.ldm;
    S.mstride = F.mstride;
    S.ksplit = F.sk_store ? 1 : F.ksplit;
    S.nquad = static_cast<int>(cq.size());
    S.qm = P.qm;
    S.qn = P.qn;
    S.c_vec = P.c_vec;
    S.r0 = static_cast<int>(r0);
    S.r1 = static_cast<int>(r1);
    S.c0 = static_cast<int>(c0);
    S.c1 = static_cast<int>(c1);
    S.mbase = F.M;
    for (size_t qi = 0; qi < cq.size(); ++qi) {
        S.cptr[qi] = cq[qi].p;
        S.crows[qi] = static_cast<int>(cq[qi].rows);
        S.ccols[qi] = static_cast<int>(cq[qi].cols);
    }
    for (size_t p = 0; p < dests.size(); ++p)
        for (const auto& [q, g] : dests[p]) {
            S.src_prod[q][S.nsrc[q]] = static_cast<int8_t>(p);
            S.src_coeff[q][S.nsrc[q]] = static_cast<int8_t>(g);
            ++S.nsrc[q];
        }
}

// Window [r0, r1) x [c0, c1) (quadrant coordinates, r0 / c0 tile multiples) of
// the plan: the mm launch over those tiles and, in split mode, the stream pass.
// wait_c() is called right before the first launch that touches C.
long run_fused_window(Engine& e, cudaStream_t s, MMParams P, const FusedPlan& F,
                      const std::vector<Terms>& dests, const std::vector<QuadView>& cq,
                      const DView& C, double alpha, long r0, long r1, long c0, long c1,
                      const std::function<void()>& wait_c) {
    // persistent launches (one CTA per SM walking the units) except where a
    // unit would take the bulk-reduction epilogue, which reuses the ring
    static const int persist_env = [] {
        const char* v = std::getenv("STRASSEN_B200_PERSISTENT");  // 0 / 1 (experiments)
        return v ? std::atoi(v) : -1;
    }();
    auto cap = [&](bool bulk_units) {
        const bool on = persist_env >= 0 ? persist_env != 0 : !bulk_units;
        return on ? (e.num_sms > 0 ? e.num_sms : 148) * (P.narrow ? 2 : 1) : 0;
    };
    const int bn = P.narrow ? kNarrowBN : kBN;
    P.tm0 = static_cast<int>(r0 / kBM);
    P.tiles_m = static_cast<int>(ceil_div(r1 - r0, kBM));
    P.tn0 = static_cast<int>(c0 / bn);
    P.tiles_n = static_cast<int>(ceil_div(c1 - c0, bn));
    if (F.tail) {
        // classical hybrid: tile owners on the first tile columns, stream-K pieces on the
        // rest (never windowed: the range is the whole output)
        FusedPlan body;  // (the plain fused plan: no tickets for a single product)
        const long split_c = static_cast<long>(F.tail_tn0) * kBN;
        long launches = run_fused_window(e, s, P, body, dests, cq, C, alpha, r0, r1, c0,
                                         std::min(c1, split_c), wait_c);
        MMParams T = P;
        T.tn0 = F.tail_tn0;
        T.tiles_n = static_cast<int>(ceil_div(c1 - split_c, kBN));
        T.mode = kEpiRMW;
        T.split = 1;
        T.ksplit = F.ksplit;
        T.kt_per_split = F.per;
        T.ldm = F.ldm;
        T.mstride = F.mstride;
        T.mbase = F.M - static_cast<long long>(split_c) * F.ldm;  // slots start at column split_c
        T.arrive = F.arrive;
        T.ticket_ld = F.ticket_ld;
        T.streamk = 1;
        T.sk_len = F.sk_len;
        T.sk_maxp = F.sk_maxp;
        T.grid_cap = F.sk_grid;  // the decode assumes exactly this many CTAs
        T.trace = trace_buffer();
        e.prof_begin("mm_kernel", s);
        ck(launch_mm(T, s), "mm_kernel (stream-K tail)");
        e.prof_end(s);
        return launches + 1;
    }
    if (!F.split) {
        wait_c();  // fused epilogue reads C
        P.mode = kEpiRMW;
        P.split = 0;
        if (F.tickets) {  // one CTA per (tile, product), C updates ordered per tile
            P.split = 1;
            P.ksplit = 1;
            P.kt_per_split = P.ktiles;
            P.tickets = F.tickets;
            P.ticket_ld = F.ticket_ld;
            static const int group_env = [] {
                const char* v = std::getenv("STRASSEN_B200_UNIT_GROUP");  // tiles (experiments)
                return v ? std::atoi(v) : 0;  // off: measured slower (r02_shortk_group.log)
            }();
            static const int group_kt = [] {
                const char* v = std::getenv("STRASSEN_B200_GROUP_KT");  // k-tiles (experiments)
                return v ? std::atoi(v) : 64;
            }();
            // Experiment (STRASSEN_B200_UNIT_GROUP=-1 auto, or G tiles): units in groups
            // of G tiles, all products of a group before the next, so a group's C
            // quadrant tiles (G x 4^L x 128 KB, ~48 MB) stay in the 126 MB L2 across
            // their ordered updates.  Measured far slower for short products
            // (profiles/r02_shortk_group.log: 16384^2 x 256 ABC L2 9.1 -> 17.3 ms,
            // 32768^2 x 1024 66.6 -> 93.1 ms): the updates of the in-flight products
            // concentrate on a few quadrant tiles and their ordered reduce-adds
            // serialise (also tried with per-(tile, quadrant) tickets).
            long g = 0;
            if (group_env >= 0) {
                g = group_env;
            } else if (P.ktiles <= group_kt) {
                const long quads = static_cast<long>(cq.size());
                g = std::max(1L, (48L << 20) / (quads * kBM * kBN * 8));
            }
            const long launch_tiles = static_cast<long>(P.tiles_m) * P.tiles_n;
            P.unit_group = g > 0 && g < launch_tiles ? static_cast<int>(g) : 0;
        }
        // bulk-reduction epilogue (C through its quadrant tensor maps); single-term
        // programs (C, DGEMM) then run persistent with a separate stage, collecting
        // each unit's reductions one unit later (kernels.cu mm_kernel, RING <
        // kRawSlots); fused-sum programs stay one CTA per unit
        const bool bulk_units = P.c_tma && P.ktiles <= P.bulk_max_kt;
        int maxt = 1;
        for (int p = 0; p < P.nprod; ++p) maxt = std::max({maxt, int{P.prod[p].na}, int{P.prod[p].nb}});
        static const bool sep_on = [] {
            const char* v = std::getenv("STRASSEN_B200_SEP");  // 0 / 1 (experiments)
            return v ? std::atoi(v) != 0 : true;
        }();
        // fused sums of <= 2 terms: persistent with the separate stage beside a 6-slot
        // ring only for short products, where the exposed per-unit epilogue outweighs
        // the shallower ring (profiles/r02_sep2_{0,1}.log: 32768^2 x 1024 ABC L2
        // 69.6 -> 64.4 ms, 16384^2 x 256 10.0 -> 8.9; but 16384^3 ABC L1 227 -> 261).
        // With product groups (longer units) only up to 8 k-tiles pays
        // (profiles/r02_sep2kt_*.log: 16384^2 x 256 ABC L2 7.18 -> 6.74 ms at 4 k-tiles,
        // but 32768^2 x 1024, 16 k-tiles, 63.1 -> 64.4)
        static const int sep2_kt = [] {
            const char* v = std::getenv("STRASSEN_B200_SEP2_KT");  // k-tiles (experiments)
            return v ? std::atoi(v) : 8;
        }();
        P.sep_stage = bulk_units && sep_on && (maxt == 1 || (maxt == 2 && P.ktiles <= sep2_kt))
                          ? 1 : 0;
        // deferred collection: the next product of a tile is tiles-in-launch units
        // later; defer only when that is >= one grid width (small host-call windows
        // would otherwise chain each tile's products one unit apart: C L2 e2e 1437 ms
        // with 16-tile windows; at 256 tiles deferral still wins, 8192^3 C L2 25.03 ->
        // 24.66 ms, the level-3 C inner calls 168.95 -> 166.5 ms)
        const long launch_tiles = static_cast<long>(P.tiles_m) * P.tiles_n;
        static const double defer_waves = [] {
            const char* v = std::getenv("STRASSEN_B200_DEFER_WAVES");  // experiments
            return v ? std::atof(v) : 1.0;
        }();
        // (grouped units: a quadrant's next update is a few products x G units later,
        // usually already running -- collect at once)
        P.sep_defer = (!F.tickets || (P.unit_group == 0 &&
                                      static_cast<double>(launch_tiles) >=
                                          defer_waves * (e.num_sms > 0 ? e.num_sms : 148)))
                          ? 1 : 0;
        P.grid_cap = cap(bulk_units && !P.sep_stage);
        if (P.grid_cap > 0) P.unit_counter = next_unit_counter(e, s);
        P.trace = trace_buffer();
        e.prof_begin("mm_kernel", s);
        ck(launch_mm(P, s), "mm_kernel");
        e.prof_end(s);
        return 1;
    }
    // cooperative fixup (kernels.hpp MMParams::coop_fixup): stream-K launches, and
    // k-chunk grids with one resident CTA per unit
    static const bool coop_on = [] {
        const char* v = std::getenv("STRASSEN_B200_COOP");  // 0 / 1 (experiments)
        return v ? std::atoi(v) != 0 : true;
    }();
    // Stream-K launches keep the single-owner fixup: sharing it measured no gain (1024^3
    // DGEMM 88.6 -> 86.7 us) or a loss (1024^3 ABC L1 90.8 -> 93.6, 1280^3 DGEMM 147.6 ->
    // 150.6: profiles/r02_cta_trace_coop_sk.log) -- every participant then also writes its own
    // partial, which the owner keeps in registers.
    static const bool coop_sk = [] {
        const char* v = std::getenv("STRASSEN_B200_COOP_SK");  // 0 / 1 (experiments)
        return v ? std::atoi(v) != 0 : false;
    }();
    if (F.fixup) {  // split mode finished by the last chunk's epilogue
        wait_c();
        P.mode = kEpiRMW;
        P.split = 1;
        P.ksplit = F.ksplit;
        P.kt_per_split = F.per;
        P.mbase = F.M;
        P.ldm = F.ldm;
        P.mstride = F.mstride;
        P.tickets = F.tickets;
        P.ticket_ld = F.ticket_ld;
        P.arrive = F.arrive;
        P.grid_cap = cap(false);
        if (F.streamk) {
            P.streamk = 1;
            P.sk_len = F.sk_len;
            P.sk_maxp = F.sk_maxp;
            P.grid_cap = F.sk_grid;  // the decode assumes exactly this many CTAs
            P.coop_fixup = coop_on && coop_sk ? 1 : 0;
        } else {
            const long units = static_cast<long>(P.tiles_m) * P.tiles_n * P.nprod * P.ksplit;
            if (coop_on && P.ksplit > 1 && P.grid_cap > 0 && units <= P.grid_cap) {
                P.coop_fixup = 1;  // one CTA per unit, all resident
                P.grid_cap = 0;
            } else if (P.grid_cap > 0) {
                P.unit_counter = next_unit_counter(e, s);
            }
        }
        // (one product: each tile takes a single update, shared by the participants)
        if (P.coop_fixup) P.tickets = nullptr;
        P.trace = trace_buffer();
        e.prof_begin("mm_kernel", s);
        ck(launch_mm(P, s), "mm_kernel (split, fused epilogue)");
        e.prof_end(s);
        return 1;
    }
    P.mode = kEpiStore;
    P.split = 1;
    P.ksplit = F.ksplit;
    P.kt_per_split = F.per;
    P.mbase = F.M;
    P.ldm = F.ldm;
    P.mstride = F.mstride;
    P.grid_cap = cap(false);
    StreamParams S;
    build_stream_params(S, P, F, dests, cq, C, alpha, r0, r1, c0, c1);
    if (F.sk_store) {  // stream-K pieces; M_p fixed up by piece 0 (kernels.cu)
        P.streamk = 1;
        P.sk_store = 1;
        P.sk_len = F.sk_len;
        P.sk_maxp = F.sk_maxp;
        P.grid_cap = F.sk_grid;  // the decode assumes exactly this many CTAs
        P.part_off = F.part_off;
        P.arrive = F.arrive;
        P.ticket_ld = F.ticket_ld;
        P.coop_fixup = coop_on && coop_sk ? 1 : 0;
    } else if (P.grid_cap > 0) {
        P.unit_counter = next_unit_counter(e, s);
    }
    P.trace = trace_buffer();
    e.prof_begin("mm_kernel", s);
    ck(launch_mm(P, s), "mm_kernel (split)");
    e.prof_end(s);
    wait_c();  // first reader of C: its copy-in overlapped the products
    e.prof_begin("stream_gather_kernel", s);
    ck(launch_stream_update(S, s), "stream_update");
    e.prof_end(s);
    return 2;
}

// Product groups for the ticketed fused-epilogue grid (MMParams::pair_mode): the
// products are reordered so that each one is followed by up to two later products
// (table order) sharing the most destination quadrants with the group; a unit then
// runs them all (the first ones parked in tensor memory) and applies alpha (g1 M1 +
// g2 M2 + g3 M3) to every destination with one update.  The level-2 table's 144 C
// updates become 90 (pairs: 109; level 1: 12 -> 7), which matters where the updates
// bound the call: short products.  Deterministic; per element the updates of a group
// are summed before they reach C (a reassociation of the reference's C + g1 M1 + g2 M2
// + g3 M3, within the BASELINE tolerance).
void pair_products(const Engine& e, MMParams& P, const FusedPlan& F, strassen_variant variant,
                   const std::vector<QuadView>& cq) {
    P.pair_mode = 0;
    static const int pair_env = [] {
        const char* v = std::getenv("STRASSEN_B200_PAIR");  // 0 / 1 / -1 auto (experiments)
        return v ? std::atoi(v) : -1;
    }();
    static const int pair_kt = [] {
        const char* v = std::getenv("STRASSEN_B200_PAIR_KT");  // k-tiles (experiments)
        // measured: 16384^2 x 256 ABC L2 9.2 -> 7.4 ms, x 1024 17.4 -> 16.8, x 4096
        // (64 k-tiles) 55.6 -> 54.9; 16384^3 (256 k-tiles) 206.0 -> 207.6 and ABC L1 at
        // x 4096 (128 k-tiles) 62.2 -> 62.4 (profiles/r02_pair12_*.log, r02_pair13_*.log)
        return v ? std::atoi(v) : 64;
    }();
    if (pair_env == 0 || F.split || !F.tickets || P.nprod < 2 || P.narrow) return;
    if (variant != STRASSEN_ABC && variant != STRASSEN_C) return;
    if (pair_env < 0 && P.ktiles > pair_kt) return;
    // (independent of C's layout and of the fused-term setting, so host and device calls
    // and every setting pair alike)
    (void)e;
    (void)cq;
    auto dests = [&](int p) {
        unsigned m = 0;
        for (int u = 0; u < P.prod[p].nc; ++u) m |= 1u << P.prod[p].cq[u];
        return m;
    };
    static const int group_max = [] {  // products per unit: 2 or 3 (kernels.cu kParkSlots + 1)
        const char* v = std::getenv("STRASSEN_B200_GROUP_MAX");  // experiments
        return v ? std::max(2, std::min(3, std::atoi(v))) : 3;
    }();
    std::vector<bool> used(static_cast<size_t>(P.nprod), false);
    std::vector<int> order;
    std::vector<int8_t> lo;
    for (int i = 0; i < P.nprod; ++i) {
        if (used[static_cast<size_t>(i)]) continue;
        used[static_cast<size_t>(i)] = true;
        lo.push_back(static_cast<int8_t>(order.size()));
        order.push_back(i);
        // grow the group with the next products (table order) sharing the most
        // destinations with it so far
        unsigned uni = dests(i);
        for (int member = 1; member < group_max; ++member) {
            int best = -1, share = 0;
            for (int j = i + 1; j < P.nprod; ++j) {
                if (used[static_cast<size_t>(j)]) continue;
                const int sh = __builtin_popcount(uni & dests(j));
                if (sh > share) {
                    share = sh;
                    best = j;
                }
            }
            if (best < 0) break;
            used[static_cast<size_t>(best)] = true;
            order.push_back(best);
            uni |= dests(best);
        }
    }
    if (static_cast<int>(lo.size()) == P.nprod) return;  // nothing shares a destination
    ProductDesc re[kMaxProducts];
    for (size_t k = 0; k < order.size(); ++k) re[k] = P.prod[order[k]];
    for (int p = 0; p < P.nprod; ++p) P.prod[p] = re[p];
    P.npairs = static_cast<int>(lo.size());
    for (int j = 0; j < P.npairs; ++j) P.pair_lo[j] = lo[static_cast<size_t>(j)];
    P.pair_lo[P.npairs] = static_cast<int8_t>(P.nprod);
    P.pair_mode = 1;
    P.a_heavy_layout = 0;  // its relayout scratch is the ring, which streams the pair's second product
    // the two products of a pair share the accumulator column map: 4 + 4-term products
    // (fully fused setting) stream whole 16-k tiles instead of half tiles
    for (int p = 0; p < P.nprod; ++p) P.prod[p].half = 0;
}

// ------------------------------------------------------------- run_device --
namespace {
long run_strassen(Engine& e, cudaStream_t s, strassen_variant variant, int level, double alpha,
                  const DView& A, const DView& B, const DView& C, const Windows* win);
long run_outer(Engine& e, cudaStream_t s, strassen_variant variant, int level, double alpha,
               const DView& A, const DView& B, const DView& C);

// Levels 0-2 run as one batched program (run_strassen); level 3 (B200
// extension) as one materialised outer level over level-2 calls (run_outer).
long run_level(Engine& e, cudaStream_t s, strassen_variant variant, int level, double alpha,
               const DView& A, const DView& B, const DView& C, const Windows* win) {
    if (variant != STRASSEN_DGEMM && level == 3) return run_outer(e, s, variant, level, alpha, A, B, C);
    return run_strassen(e, s, variant, level, alpha, A, B, C, win);
}

// Device memory new temporaries may take: free memory less a margin of 4% of the
// device (allocation granularity, ticket buffers, other libraries' small
// allocations).  STRASSEN_B200_MEM_CAP overrides it (tests / experiments).
double device_bytes_free(void) {
    if (const char* cap = std::getenv("STRASSEN_B200_MEM_CAP")) return std::atof(cap);
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return 1e300;
    }
    return static_cast<double>(free_b) -
           std::max(0.04 * static_cast<double>(total_b), static_cast<double>(2ULL << 30));
}

DView sub(const DView& v, long r0, long c0, long rows, long cols) {
    DView o = v;
    o.p = v.p + r0 * v.rs + c0 * v.cs;
    o.rows = rows;
    o.cols = cols;
    return o;
}
}  // namespace

std::vector<int> window_order(int rows, int cols) {
    std::vector<int> order;
    for (int sh = 0; sh < std::max(rows, cols); ++sh) {
        if (sh < cols)
            for (int r = 0; r < std::min(sh, rows); ++r) order.push_back(r * cols + sh);
        if (sh < rows)
            for (int c = 0; c <= std::min(sh, cols - 1); ++c) order.push_back(sh * cols + c);
    }
    return order;
}

void plan_windows(const Engine& e, strassen_variant variant, int level, long m, long n, long k,
                  bool row_windows, Windows& w) {
    (void)k;
    w.rows = w.cols = 0;
    const int L = (variant == STRASSEN_DGEMM) ? 0 : level;
    if (L > 2) return;  // level 3: the outer level runs whole-operand (run_outer)
    const long side = 1L << L;
    const long qm = ceil_div(m, side), qn = ceil_div(n, side);
    const long tiles_m = ceil_div(qm, kBM), tiles_n = ceil_div(qn, kBN);
    const long sms = e.num_sms > 0 ? e.num_sms : 148;
    // CTAs per output tile: one per product (AB / Naive store products; ABC / C
    // run the ticketed (tile, product) grid), one for DGEMM
    long per_tile = 1;
    for (int l = 0; l < L; ++l) per_tile *= 7;
    if (variant != STRASSEN_NAIVE && variant != STRASSEN_AB && tiles_m * tiles_n < 2 * sms)
        return;  // split-mode sizes: a few milliseconds, nothing to overlap
    {   // temporaries that need product groups (run_strassen) rule out windows
        const long qk = ceil_div(k, side);
        // materialised sums per side of the full tables: every multi-term side
        // (Naive, C; ABC / AB fusing single terms only), or the sides longer than
        // the fused limit (level 2's 25 four-term sides)
        const bool all = variant == STRASSEN_NAIVE || variant == STRASSEN_C ||
                         (variant != STRASSEN_DGEMM && e.fuse_max_terms < 2);
        const double nsums = all ? (L == 1 ? 5.0 : 45.0)
                             : (variant != STRASSEN_DGEMM && L == 2 && e.fuse_max_terms < 4) ? 25.0
                                                                                             : 0.0;
        const double sums = nsums * 8.0 * (qm * qk + qk * qn);
        const double prods = (variant == STRASSEN_NAIVE || variant == STRASSEN_AB)
                                 ? per_tile * 8.0 * qm * qn : 0.0;
        const double held = static_cast<double>(e.tabuf.bytes + e.tbbuf.bytes + e.mbuf.bytes);
        if (sums + prods > held && sums + prods > device_bytes_free() + held) return;
    }
    // windows of >= 2 waves each (consecutive windows overlap on two streams);
    // grow the grid keeping it square-ish
    const long max_w = tiles_m * tiles_n * per_tile / (2 * sms);
    constexpr long kUniform = 8;  // uniform strips per side
    long R = 1, Cn = 1;
    for (;;) {
        const bool grow_c = Cn < kUniform && Cn < tiles_n && R * (Cn + 1) <= max_w;
        const bool grow_r = row_windows && R < kUniform && R < tiles_m &&
                            (R + 1) * Cn <= max_w;
        if (grow_c && (Cn <= R || !grow_r)) ++Cn;
        else if (grow_r) ++R;
        else break;
    }
    if (const char* env = std::getenv("STRASSEN_B200_WINDOWS")) {  // "RxC" (experiments)
        long r = 0, c = 0;
        if (std::sscanf(env, "%ldx%ld", &r, &c) == 2) {
            R = clip(r, 1, row_windows ? std::min<long>(Engine::kMaxStrips, tiles_m) : 1);
            Cn = clip(c, 1, std::min<long>(Engine::kMaxStrips, tiles_n));
        }
    }
    if (R * Cn < 2) return;
    // Strips of equal width, the first one replaced by a ramp 1, 1, 2, 4, ... tiles:
    // the first windows need only a sliver of A and B, so compute starts after
    // ~1/16 of the transfer time instead of ~1/4 (windows stay small at the end,
    // where each one's copy-back is exposed).
    // optional ramp (experiments): STRASSEN_B200_RAMP="1,1,2" splits the first
    // strip into those tile counts
    std::vector<long> ramp;
    if (const char* rs = std::getenv("STRASSEN_B200_RAMP")) {
        for (const char* c = rs; *c;) {
            char* end = nullptr;
            const long v = std::strtol(c, &end, 10);
            if (end == c) break;
            if (v > 0) ramp.push_back(v);
            c = (*end == ',') ? end + 1 : end;
        }
    }
    auto bounds = [&](long tiles, long count, long q) {
        const long u = ceil_div(tiles, count);
        std::vector<long> sizes;
        long left = u;
        for (long r : ramp) {
            if (left <= 0) break;
            sizes.push_back(std::min(r, left));
            left -= sizes.back();
        }
        if (left > 0) sizes.push_back(left);
        for (long t = u; t < tiles; t += u) sizes.push_back(std::min(u, tiles - t));
        std::vector<long> b{0};
        for (long sz : sizes) b.push_back(std::min(q, b.back() + sz * kBM));
        b.back() = q;
        return b;
    };
    w.rb = bounds(tiles_m, R, qm);
    w.cb = bounds(tiles_n, Cn, qn);
    if (static_cast<long>(w.rb.size()) - 1 > Engine::kMaxStrips ||
        static_cast<long>(w.cb.size()) - 1 > Engine::kMaxStrips)
        return;  // too many strips for the event pools: keep the unwindowed call
    w.rows = static_cast<int>(w.rb.size()) - 1;
    w.cols = static_cast<int>(w.cb.size()) - 1;
}

// Dynamic peeling (north star; the reference pads instead, matrix.cpp:14-22):
// when m, n or k is not a multiple of 2^L, Strassen runs on the even core
// m_e x n_e x k_e (every quadrant full, no padded tiles) and three classical
// fringe updates finish the product:
//   C[0:m_e, 0:n_e] += alpha A[0:m_e, k_e:k] B[k_e:k, 0:n_e]   (rank-k_r)
//   C[m_e:m, 0:n]   += alpha A[m_e:m, 0:k]   B                  (bottom rows)
//   C[0:m_e, n_e:n] += alpha A[0:m_e, 0:k]   B[0:k, n_e:n]      (right columns)
// Tiny problems (core below one 128-tile per quadrant) keep the padded path.
long run_device(Engine& e, cudaStream_t s, strassen_variant variant, int level, double alpha,
                const DView& A, const DView& B, const DView& C, const Windows* win) {
    const int L = (variant == STRASSEN_DGEMM) ? 0 : level;
    const long S = 1L << L;
    const long m = A.rows, k = A.cols, n = B.cols;
    // Dynamic peeling: the core is the largest problem with dimensions that are multiples
    // of 2^L -- or, where a dimension exceeds a whole number of quadrant tiles by at most
    // the fringe kernels' width (4100 at level 2: quadrants of 1025 = 8 tiles + 1 row,
    // which would run a ninth, padded tile row), the multiple of 2^L x 128 below it.
    auto core = [&](long d, long tile) { return peel_core(d, S, tile, fringe_max_width()); };
    static const bool tile_peel = [] {
        const char* v = std::getenv("STRASSEN_B200_TILE_PEEL");  // 0 / 1 (experiments)
        return v ? std::atoi(v) != 0 : true;
    }();
    // (not for a pipelined host call: a peeled call cannot run in windows, and losing the
    // transfer overlap costs more than the padded tiles -- it keeps the multiple-of-2^L
    // rule, so at these shapes it rounds differently from the device call)
    const bool windowed = win && win->count() > 0;
    const long me = tile_peel && !windowed ? core(m, kBM) : m & ~(S - 1);
    const long ne = tile_peel && !windowed ? core(n, kBN) : n & ~(S - 1);
    const long ke = k & ~(S - 1);
    const bool ragged = me != m || ne != n || ke != k;
    // peel only when it removes padded work: compare output-tile x k-step counts
    auto work = [&](long mm, long nn, long kk) {
        return ceil_div(ceil_div(mm, S), kBM) * ceil_div(ceil_div(nn, S), kBN) *
               ceil_div(ceil_div(kk, S), kBK);
    };
    const bool peel = ragged && e.peeling && me >= S * kBM && ne >= S * kBN && ke >= S * kBK &&
                      m - me <= fringe_max_width() && n - ne <= fringe_max_width() &&
                      (L > 0 || tile_peel) &&
                      peel_pays(work(m, n, k), work(me, ne, ke), L == 0 ? 1 : L == 1 ? 7 : L == 2 ? 49 : 343,
                                e.num_sms > 0 ? e.num_sms : 148, fringe_bytes(m, n, k, me, ne, ke));
    if (win && win->count() > 0 &&
        (peel || !tma_ready(A, ceil_div(m, S), static_cast<int>(S)) ||
         !tma_ready(B, ceil_div(k, S), static_cast<int>(S)))) {
        // not windowable: everything in first, everything out last
        for (int r = 0; r < win->rows; ++r) win->issue_a(r);
        for (int c = 0; c < win->cols; ++c) win->issue_b(c);
        for (int w = 0; w < win->count(); ++w) win->issue_c(w);
        for (int r = 0; r < win->rows; ++r) ck(cudaStreamWaitEvent(s, win->a_ready[r], 0), "wait");
        for (int c = 0; c < win->cols; ++c) ck(cudaStreamWaitEvent(s, win->b_ready[c], 0), "wait");
        for (int w = 0; w < win->count(); ++w)
            ck(cudaStreamWaitEvent(s, win->c_ready[w], 0), "wait");
        const long launches = run_device(e, s, variant, level, alpha, A, B, C, nullptr);
        for (int w = 0; w < win->count(); ++w) {
            ck(cudaEventRecord(win->done[w], s), "window done");
            win->issue_out(w);
        }
        return launches;
    }
    if (!peel) return run_level(e, s, variant, level, alpha, A, B, C, win);
    long launches = run_level(e, s, variant, level, alpha, sub(A, 0, 0, me, ke),
                              sub(B, 0, 0, ke, ne), sub(C, 0, 0, me, ne), nullptr);
    // The three fringe updates (at most 2^L - 1 wide): streaming kernels (fringe.cu) --
    // through the tile kernel a 1 x 4097 x 4097 update ran 33 CTAs over the whole k
    // loop, 0.5 ms of the 4.3 ms call.  STRASSEN_B200_FRINGE=0: the tile kernel.
    static const bool fringe_on = [] {
        const char* v = std::getenv("STRASSEN_B200_FRINGE");  // 0 / 1 (experiments)
        return v ? std::atoi(v) != 0 : true;
    }();
    const bool thin = fringe_on && S - 1 <= fringe_max_width();
    if (thin) {  // (operands still being copied in: the core has waited on s already)
        wait_ready(s, A);
        wait_ready(s, B);
        wait_ready(s, C);
    }
    auto part = [&](long long_len, long thin_w, long kk) {
        return e.ensure(e.fringe_buf, fringe_partial_bytes(long_len, static_cast<int>(thin_w), kk));
    };
    if (ke < k) {
        const DView a = sub(A, 0, ke, me, k - ke), b = sub(B, ke, 0, k - ke, ne);
        const DView c = sub(C, 0, 0, me, ne);
        if (thin) {
            e.prof_begin("fringe_k_kernel", s);
            ck(launch_fringe_k(a.p, a.rs, a.cs, b.p, b.rs, b.cs, c.p, c.rs, c.cs, me, ne,
                               static_cast<int>(k - ke), alpha, s),
               "fringe (k)");
            e.prof_end(s);
            ++launches;
        } else {
            launches += run_strassen(e, s, STRASSEN_DGEMM, 0, alpha, a, b, c, nullptr);
        }
    }
    if (me < m) {
        const DView a = sub(A, me, 0, m - me, k), c = sub(C, me, 0, m - me, n);
        if (thin) {
            double* w = part(n, m - me, k);
            int nkc = 0;
            e.prof_begin("fringe_m_kernel", s);
            ck(launch_fringe_m(a.p, a.rs, a.cs, B.p, B.rs, B.cs, static_cast<int>(m - me), n, k,
                               w, &nkc, s),
               "fringe (m)");
            e.prof_end(s);
            e.prof_begin("fringe_reduce_kernel", s);
            ck(launch_fringe_reduce(w, nkc, static_cast<int>(m - me), n, alpha, c.p, c.cs, c.rs, s),
               "fringe (m) reduce");
            e.prof_end(s);
            launches += 2;
        } else {
            launches += run_strassen(e, s, STRASSEN_DGEMM, 0, alpha, a, B, c, nullptr);
        }
    }
    if (ne < n) {
        const DView a = sub(A, 0, 0, me, k), b = sub(B, 0, ne, k, n - ne);
        const DView c = sub(C, 0, ne, me, n - ne);
        if (thin) {
            double* w = part(me, n - ne, k);
            int nkc = 0;
            e.prof_begin("fringe_n_kernel", s);
            ck(launch_fringe_n(a.p, a.rs, a.cs, b.p, b.rs, b.cs, me, static_cast<int>(n - ne), k,
                               w, &nkc, s),
               "fringe (n)");
            e.prof_end(s);
            e.prof_begin("fringe_reduce_kernel", s);
            ck(launch_fringe_reduce(w, nkc, static_cast<int>(n - ne), me, alpha, c.p, c.rs, c.cs, s),
               "fringe (n) reduce");
            e.prof_end(s);
            launches += 2;
        } else {
            launches += run_strassen(e, s, STRASSEN_DGEMM, 0, alpha, a, b, c, nullptr);
        }
    }
    return launches;
}

namespace {
long run_strassen(Engine& e, cudaStream_t s, strassen_variant variant, int level, double alpha,
                  const DView& A, const DView& B, const DView& C, const Windows* win) {
    const int L = (variant == STRASSEN_DGEMM) ? 0 : level;
    const int side = 1 << L;
    const long m = A.rows, k = A.cols, n = B.cols;
    const long qm = ceil_div(m, side), qk = ceil_div(k, side), qn = ceil_div(n, side);
    long launches = 0;
    const TmaOperand ta = prepare(e, s, A, qm, qk, side, e.pack_a, launches);
    const TmaOperand tb = prepare(e, s, B, qk, qn, side, e.pack_b, launches);
    const int nq = side * side;
    std::vector<bool> a_live(nq), b_live(nq), c_live(nq);
    std::vector<QuadView> cq(nq);
    for (int I = 0; I < side; ++I)
        for (int J = 0; J < side; ++J) {
            a_live[I * side + J] = quad_rows(ta, I) > 0 && quad_cols(ta, J) > 0;
            b_live[I * side + J] = quad_rows(tb, I) > 0 && quad_cols(tb, J) > 0;
            cq[I * side + J] = c_quad(C, qm, qn, I, J);
            c_live[I * side + J] = cq[I * side + J].rows > 0 && cq[I * side + J].cols > 0;
        }

    MMParams P;
    std::memset(&P, 0, sizeof(P));
    // Narrow tiles (kernels.hpp kNarrowBN: 128 x 64, two CTAs per SM) for small
    // single-term programs: a CTA's fixed costs (pipeline fill, fixup, epilogue) then
    // overlap the other CTA's mainloop.  Measured (profiles/r02_narrow_sweep.log,
    // back-to-back us wide -> narrow): DGEMM 1024^3 90.5 -> 86.8, 768^3 61.4 -> 57.1;
    // C L2 1024^3 130.9 -> 126.9, 1280^3 228.1 -> 208.8, 2048^3 570.0 -> 532.7, 2560^3
    // 989.8 -> 943.2; C L1 1280^3 158.3 -> 154.9; neutral to slower from 1536^3
    // (DGEMM) / 3072^3 (C L2).  Fused-sum programs (ABC, AB) lose (1024^3 ABC L1
    // 89.9 -> 94.3: a fused k-step streams 1.5x the operand bytes per flop) and keep
    // 128 x 128 tiles.  Naive stays under the 4 waves from which host calls run in
    // windows (plan_windows), so host and device calls plan alike.  Decided on the
    // problem alone (not on the fused-term setting, which must not change a bit).
    {
        static const int narrow_env = [] {
            const char* v = std::getenv("STRASSEN_B200_NARROW");  // 0 / 1 / -1 auto (experiments)
            return v ? std::atoi(v) : -1;
        }();
        const long sms = e.num_sms > 0 ? e.num_sms : 148;
        const long tiles = ceil_div(qm, kBM) * ceil_div(qn, kBN);
        const long units = tiles * (L == 0 ? 1 : L == 1 ? 7 : 49);
        const long ktiles = ceil_div(qk, kBK);
        const bool one_window = !win || win->rows * win->cols <= 1;
        // A quadrant whose last 128-wide tile column is at most half used (2816^3 at
        // level 2: quadrants of 704 = 5.5 tiles) wastes less on 64-wide tiles: C / Naive
        // L2 2816^3 32.6 -> 35.0 TF/s, 3840^3 35.3 -> 38.1, 4864^3 37.8 -> 40.1, 6400^3
        // 40.0 -> 40.5 (profiles/r02_narrow_half_edge.log).  At these sizes the programs
        // split nothing in k, so narrow and wide tiles give bitwise the same result
        // (tools/narrow_check.py) and windowed host calls may keep the wide tiles.
        const long rem_n = qn % kBN;
        const bool half_edge = rem_n > 0 && rem_n <= kNarrowBN && ceil_div(qn, kBN) <= 15;
        bool pick = false;
        if (ktiles <= 128) {
            if (variant == STRASSEN_DGEMM) pick = 3 * tiles < 2 * sms;
            else if (variant == STRASSEN_C) pick = units < 10 * sms || half_edge;
            else if (variant == STRASSEN_NAIVE) pick = units < 4 * sms || half_edge;
            // AB at level 2 (its 4-term sides are materialised, the rest are 2-term sums:
            // the narrow kernel's limit) gains there too -- 3840^3 34.4 -> 36.5 TF/s, 4864^3
            // 36.8 -> 38.2 -- and stores products like Naive, so the result is bitwise the
            // wide one; at level 1 the gain is ~2% and ABC keeps its grouped epilogue
            else if (variant == STRASSEN_AB && L == 2 && e.fuse_max_terms <= 2) pick = half_edge;
        }
        P.narrow = one_window && (narrow_env > 0 || (narrow_env < 0 && pick)) ? 1 : 0;
    }
    const int bn = P.narrow ? kNarrowBN : kBN;
    for (int I = 0; I < side; ++I)
        for (int J = 0; J < side; ++J) {
            const int qi = I * side + J;
            if (a_live[qi])
                encode_map(&P.tmA[qi], quad_origin(ta, I, J), quad_rows(ta, I), quad_cols(ta, J),
                           ta.ld, 16, kBK, 128);
            if (b_live[qi])
                encode_map(&P.tmB[qi], quad_origin(tb, I, J), quad_rows(tb, I), quad_cols(tb, J),
                           tb.ld, kBK, bn, 128);
            if (L == 2 && a_live[qi] && !P.narrow)  // half-k maps for the (4,4) products
                encode_map(&P.tmAh[qi], quad_origin(ta, I, J), quad_rows(ta, I),
                           quad_cols(ta, J), ta.ld, 16, kBK / 2, 128);
            if (L == 2 && b_live[qi] && !P.narrow)
                encode_map(&P.tmBh[qi], quad_origin(tb, I, J), quad_rows(tb, I),
                           quad_cols(tb, J), tb.ld, kBK / 2, kBN, 64);
            P.cptr[qi] = cq[qi].p;
            P.crows[qi] = static_cast<int>(cq[qi].rows);
            P.ccols[qi] = static_cast<int>(cq[qi].cols);
        }
    P.rs_c = C.rs;
    P.cs_c = C.cs;
    P.alpha = alpha;
    {   // 16-byte epilogue: C column-major, even ldc, every quadrant origin aligned
        bool vec = C.rs == 1 && C.cs % 2 == 0 && (reinterpret_cast<uintptr_t>(C.p) % 16) == 0;
        for (int qi = 0; qi < side * side && vec; ++qi)
            vec = (reinterpret_cast<uintptr_t>(cq[qi].p) % 16) == 0;
        P.c_vec = vec ? 1 : 0;
        // C quadrant tensor maps for the bulk-reduction epilogue: 16-row x
        // 128-column boxes, 128-byte swizzle, one TMA reduce-add per box
        if (vec && C.cs * 8 < (1LL << 40) && !P.narrow) {  // (narrow: register epilogues)
            for (int qi = 0; qi < side * side; ++qi)
                if (c_live[qi])
                    encode_map(&P.tmC[qi], cq[qi].p, cq[qi].rows, cq[qi].cols, C.cs, 16, kBN, 128);
            P.c_tma = 1;
        }
    }
    P.qm = static_cast<int>(qm);
    P.qn = static_cast<int>(qn);
    P.qk = static_cast<int>(qk);
    P.tiles_m = static_cast<int>(ceil_div(qm, kBM));
    P.tiles_n = static_cast<int>(ceil_div(qn, bn));
    P.ktiles = static_cast<int>(ceil_div(qk, kBK));
    P.group_m = 8;
    // bulk-reduction epilogue (C tiles staged in smem, one TMA reduce-add per
    // 16 x 128 box) at every k: with the tensor-map reduce-adds and the deferred
    // completion of persistent single-term launches it beats the register
    // read-modify-write everywhere measured (16384^3: C L2 196.5 -> 190.6 ms,
    // DGEMM 246.9 -> 242.5, ABC L2 239.7 -> 235.9; profiles/r01_bulk_kt_probe.log)
    P.bulk_max_kt = 1 << 30;
    {
        static const bool lay1 = [] {
            const char* v = std::getenv("STRASSEN_B200_LAYOUT1");  // 0 / 1 (experiments)
            return v ? std::atoi(v) != 0 : true;
        }();
        P.a_heavy_layout = lay1 ? 1 : 0;
    }
    if (const char* b = std::getenv("STRASSEN_B200_BULK_MAX_KT")) P.bulk_max_kt = std::atoi(b);

    // Live products in table order (variants.cpp:130-133 skip rule).
    struct Live {
        Terms a, b, c;
    };
    std::vector<Live> live;
    // profiling aid only (wrong results): keep the products with "na,nb" terms
    static const int only_combo = [] {
        const char* v = std::getenv("STRASSEN_B200_PROFILE_ONLY_COMBO");
        int na = 0, nb = 0;
        return v && std::sscanf(v, "%d,%d", &na, &nb) == 2 ? na * 8 + nb : 0;
    }();
    for (const Product& pr : program(L).products) {
        Live l{live_terms(pr.a, a_live), live_terms(pr.b, b_live), live_terms(pr.c, c_live)};
        if (l.a.empty() || l.b.empty() || l.c.empty()) continue;
        if (only_combo && static_cast<int>(l.a.size() * 8 + l.b.size()) != only_combo) continue;
        live.push_back(std::move(l));
    }
    // The whole program, or -- when the materialised operand sums and product
    // temporaries of all live products would not fit in device memory (Naive / C /
    // AB at very large sizes) -- consecutive groups of products in table order, each
    // with its own sum pass, products and C updates.  Every C element still receives
    // its updates in table order.
    // the whole program's size and mean term count plan every group's launches
    // Operand sides with at least mat_min terms are materialised by the sum pass
    // (materialize_sum, variants.cpp:53-96); shorter ones are summed in the mm
    // kernel's registers (pack_a_sum / pack_b_sum, blocking.cpp:12-66).  Naive and
    // C materialise every multi-term side; ABC and AB fuse sides of up to
    // e.fuse_max_terms terms.  Both forms add the terms in listed order with the
    // same roundings, so the choice never changes a bit of the result.
    const int mat_min_f = (variant == STRASSEN_C || variant == STRASSEN_NAIVE) ? 2
                        : (variant == STRASSEN_DGEMM)                        ? kMaxTerms + 1
                                                                             : e.fuse_max_terms + 1;
    // (narrow-tile kernels sum at most 2 terms per side: longer sides are materialised,
    // bitwise the same as summing them in registers)
    const int mat_min = P.narrow ? std::min(mat_min_f, 3) : mat_min_f;
    // The launch plan (k-chunks, stream-K pieces) must not depend on where the sums
    // are formed, or the fused-term setting would change roundings: it is made for the
    // variant's own term counts (ABC / AB as fully fused, Naive / C single-term).
    const bool fusing = variant == STRASSEN_ABC || variant == STRASSEN_AB;
    const int nprod_all = static_cast<int>(live.size());
    double terms_all = 0.0;
    for (const Live& l : live)
        terms_all += fusing ? 0.5 * static_cast<double>(l.a.size() + l.b.size()) : 1.0;
    terms_all /= std::max(1, nprod_all);
    auto run_program = [&](std::vector<Live> live, MMParams P) -> long {
        // Windows (r, c) in row-major order; without `win` one window covers all.
        const int nr = win ? win->rows : 1, nc = win ? win->cols : 1, nw = nr * nc;

        // Windows alternate between s and the aux stream (ordered after s's work so
        // far); s joins the aux stream at the end.
        cudaStream_t ws[2] = {s, nw > 1 ? e.aux_stream : s};
        auto wait_ev = [&](cudaStream_t st, cudaEvent_t ev) {
            if (ev) ck(cudaStreamWaitEvent(st, ev, 0), "wait");
        };
        auto wait_a = [&](cudaStream_t st, int r) { wait_ev(st, win ? win->a_ready[r] : ta.ready); };
        auto wait_b = [&](cudaStream_t st, int c) { wait_ev(st, win ? win->b_ready[c] : tb.ready); };
        auto wait_c = [&](cudaStream_t st, int w) {
            if (win) wait_ev(st, win->c_ready[w]);
            else wait_ready(st, C);
        };
        auto finish = [&](cudaStream_t st, int w) {
            if (!win) return;
            ck(cudaEventRecord(win->done[w], st), "window done");
            win->issue_out(w);
        };
        // processing order; the first window of each row strip computes its A
        // sums (and triggers its copy), likewise for column strips and B
        const std::vector<int> order = win ? window_order(nr, nc) : std::vector<int>{0};
        std::vector<int> first_r(nr, -1), first_c(nc, -1);
        for (int i = 0; i < nw; ++i) {
            if (first_r[order[i] / nc] < 0) first_r[order[i] / nc] = order[i];
            if (first_c[order[i] % nc] < 0) first_c[order[i] % nc] = order[i];
        }
        auto prefetch = [&](int i) {  // copies of the i-th window, issued one window ahead
            if (!win || i >= nw) return;
            const int w = order[i], r = w / nc, c = w % nc;
            if (first_r[r] == w) win->issue_a(r);
            if (first_c[c] == w) win->issue_b(c);
            win->issue_c(w);
        };
        auto join = [&] {
            if (nw > 1) {
                ck(cudaEventRecord(e.ev_join, e.aux_stream), "join");
                ck(cudaStreamWaitEvent(s, e.ev_join, 0), "join");
            }
        };

        prefetch(0);
        if (live.empty()) {
            for (int i = 0; i < nw; ++i) {
                prefetch(i + 1);
                wait_c(s, order[i]);
                finish(s, order[i]);
            }
            join();
            return launches;
        }

        bool sums = false;
        for (const Live& l : live)
            sums = sums || l.a.size() >= static_cast<size_t>(mat_min) ||
                   l.b.size() >= static_cast<size_t>(mat_min);
        std::unique_ptr<SumBatchParams> side_sums[2];
        if (sums) {
            // Every multi-term operand sum materialised by one HBM pass per side
            // (materialize_sum, variants.cpp:53-96, for all entries at once); the
            // mm launch then runs all 7^L products with single-term operands.
            //   C variant (B200 addition): fused multi-destination epilogue.
            //   Naive: products to temporaries M_p, then one stream pass applying
            //          C_r += alpha*gamma*M_p in table order (variants.cpp:99-109).
            const long long lda_t = ((qm + 3) / 4) * 4, ldb_t = ((qk + 3) / 4) * 4;
            int na_sums = 0, nb_sums = 0;
            for (const Live& l : live) {
                na_sums += l.a.size() >= static_cast<size_t>(mat_min);
                nb_sums += l.b.size() >= static_cast<size_t>(mat_min);
            }
            double* TA = e.ensure(e.tabuf, static_cast<size_t>(std::max(na_sums, 1)) * lda_t * qk * 8);
            double* TB = e.ensure(e.tbbuf, static_cast<size_t>(std::max(nb_sums, 1)) * ldb_t * qn * 8);
            for (int sd = 0; sd < 2; ++sd) {
                side_sums[sd].reset(new SumBatchParams);  // ~10 KB: keep off the stack
                SumBatchParams* SB = side_sums[sd].get();
                std::memset(SB, 0, sizeof(*SB));
                int next_map = kMaxQuad;  // tmA / tmB: 16 quadrant maps, then the sums
                const TmaOperand& t = sd == 0 ? ta : tb;
                SB->rows = sd == 0 ? qm : qk;
                SB->cols = sd == 0 ? qk : qn;
                SB->ld = sd == 0 ? lda_t : ldb_t;
                for (size_t p = 0; p < live.size(); ++p) {
                    Terms& terms = sd == 0 ? live[p].a : live[p].b;
                    // fused in the kernel: the quadrant maps, signs in-kernel
                    if (terms.size() < static_cast<size_t>(mat_min)) continue;
                    const int z = SB->njobs++;
                    double* dst = (sd == 0 ? TA : TB) + static_cast<size_t>(z) * SB->ld * SB->cols;
                    SB->dst[z] = dst;
                    SB->nterms[z] = static_cast<int>(terms.size());
                    for (size_t u = 0; u < terms.size(); ++u) {
                        const int qi = terms[u].first;
                        SumTerm& st = SB->t[z][u];
                        st.x = quad_origin(t, qi / side, qi % side);
                        st.rows = static_cast<int>(quad_rows(t, qi / side));
                        st.cols = static_cast<int>(quad_cols(t, qi % side));
                        st.ld = t.ld;
                        st.coeff = terms[u].second;
                    }
                    const int mi = next_map++;
                    if (mi >= kMaxMaps) throw Error(STRASSEN_ERR_PARAM, "too many operand maps");
                    if (sd == 0)
                        encode_map(&P.tmA[mi], dst, qm, qk, lda_t, 16, kBK, 128);
                    else
                        encode_map(&P.tmB[mi], dst, qk, qn, ldb_t, kBK, bn, 128);
                    terms = {{mi, 1}};
                }
            }
        }

        // First A and B terms at +1 (kernels.cu product_kloop): a side whose first
        // coefficient is -1 is negated as a whole, and so are the destination
        // coefficients.  Exact: (-S) x T = -(S x T) bit for bit under round-to-nearest.
        for (Live& l : live)
            for (Terms* t : {&l.a, &l.b})
                if (t->front().second < 0) {
                    for (auto& x : *t) x.second = -x.second;
                    for (auto& x : l.c) x.second = -x.second;
                }

        P.nprod = static_cast<int>(live.size());
        std::vector<Terms> dests;
        for (size_t p = 0; p < live.size(); ++p) {
            fill_desc(P.prod[p], live[p].a, live[p].b, live[p].c);
            dests.push_back(live[p].c);
        }
        // C / ABC / DGEMM: fused epilogue (split only when few tiles).  AB, Naive:
        // products to temporaries on a product-parallel grid (one CTA per tile x
        // product: balanced waves at every size), then one stream pass
        // (AB: variants.cpp:142-168).
        const bool store_products = variant == STRASSEN_NAIVE || variant == STRASSEN_AB;
        const FusedPlan F = plan_fused(e, s, P, store_products, nprod_all, terms_all, nw > 1);
        pair_products(e, P, F, variant, cq);
        if (nw > 1) {  // the aux stream starts after everything enqueued on s so far
            ck(cudaEventRecord(e.ev_fork, s), "fork");
            ck(cudaStreamWaitEvent(e.aux_stream, e.ev_fork, 0), "fork");
        }

        for (int i = 0; i < nw; ++i) {
            prefetch(i + 1);
            const int w = order[i], r = w / nc, c = w % nc;
            cudaStream_t st = ws[i % 2];
            const long r0 = win ? win->rb[r] : 0, r1 = win ? win->rb[r + 1] : qm;
            const long c0 = win ? win->cb[c] : 0, c1 = win ? win->cb[c + 1] : qn;
            wait_a(st, r);
            wait_b(st, c);
            if (sums) {
                // A sums of row strip r in its first window, B sums of column strip c
                // in row 0; later windows wait on them
                for (int sd = 0; sd < 2; ++sd) {
                    SumBatchParams& SB = *side_sums[sd];
                    const bool owner = sd == 0 ? first_r[r] == w : first_c[c] == w;
                    cudaEvent_t ev = sd == 0 ? e.ev_sum_a[r] : e.ev_sum_b[c];
                    if (!owner) {
                        wait_ev(st, ev);
                        continue;
                    }
                    if (!SB.njobs) continue;
                    if (sd == 0) {
                        SB.r0 = r0;
                        SB.rows = r1;
                    } else {
                        SB.c0 = c0;
                        SB.cols = c1;
                    }
                    e.prof_begin("sum_gather_kernel", st);
                    ck(launch_sum_batch(SB, st), sd == 0 ? "sum_batch (A)" : "sum_batch (B)");
                    e.prof_end(st);
                    ++launches;
                    if (nw > 1) ck(cudaEventRecord(ev, st), "sum event");
                }
            }
            launches += run_fused_window(e, st, P, F, dests, cq, C, alpha, r0, r1, c0, c1,
                                         [&] { wait_c(st, w); });
            finish(st, w);
        }
        join();
        return launches;
    };
    int n_as = 0, n_bs = 0;
    for (const Live& l : live) {
        n_as += l.a.size() >= static_cast<size_t>(mat_min);
        n_bs += l.b.size() >= static_cast<size_t>(mat_min);
    }
    const bool sums_v = n_as + n_bs > 0;
    const bool store_v = variant == STRASSEN_NAIVE || variant == STRASSEN_AB;
    const double a_sum = 8.0 * (((qm + 3) / 4) * 4) * qk, b_sum = 8.0 * (((qk + 3) / 4) * 4) * qn;
    const double m_tmp = 8.0 * ((qm + 1) / 2 * 2) * qn;
    // temporaries per live product (each side allocates at least one sum slot, so a
    // single-term side counts as a sum too)
    auto need = [&](size_t) { return (sums_v ? a_sum + b_sum : 0.0) + (store_v ? m_tmp : 0.0); };
    // the one-shot program's buffers against what the ctx already holds
    const double need_a = sums_v ? std::max(n_as, 1) * a_sum : 0.0;
    const double need_b = sums_v ? std::max(n_bs, 1) * b_sum : 0.0;
    const double need_m = store_v ? static_cast<double>(live.size()) * m_tmp : 0.0;
    const double extra = std::max(0.0, need_a - static_cast<double>(e.tabuf.bytes)) +
                         std::max(0.0, need_b - static_cast<double>(e.tbbuf.bytes)) +
                         std::max(0.0, need_m - static_cast<double>(e.mbuf.bytes));
    // (cudaMemGetInfo only when the buffers must grow: on the hot path it stalled
    // calls by up to ~80 ms now and then -- profiles/r01_notes.md)
    if (win || live.size() <= 1 || extra <= 0.0 || extra <= device_bytes_free())
        return run_program(live, P);
    // Not enough: give the ctx's temporaries back and run groups that fit
    if (e.capturing)
        throw Error(STRASSEN_ERR_ALLOC, "stream capture: the call's temporaries do not fit "
                                        "beside the ctx's workspace (product groups release it)");
    ck(cudaDeviceSynchronize(), "sync before releasing temporaries");
    for (DeviceBuffer* b : {&e.tabuf, &e.tbbuf, &e.mbuf})
        if (b->ptr) {
            cudaFree(b->ptr);
            b->ptr = nullptr;
            b->bytes = 0;
        }
    const double avail = device_bytes_free();
    size_t i0 = 0;
    while (i0 < live.size()) {
        size_t i1 = i0 + 1;
        double t = need(i0);
        while (i1 < live.size() && t + need(i1) <= avail) t += need(i1++);
        std::vector<Live> group(live.begin() + static_cast<long>(i0), live.begin() + static_cast<long>(i1));
        run_program(group, P);
        i0 = i1;
    }
    return launches;
}
}  // namespace

namespace {
// Level 3 for the materialising variants (Naive, C) -- a B200 extension: the
// reference composes level-3 tables symbolically (table.cpp:47-67,
// acceptance.cpp:86-88) but its runtime stops at level 2 (table.cpp:101).
// Level 3 = the one-level table (table.cpp:18-33) applied with Naive semantics
// (variants.cpp:170-208) over level-2 calls of the same variant:
//   1. every outer operand sum S_r = sum_u c_u X_{q_u} (quadrants of the even
//      ceil partition, matrix.cpp:8-35; clipped terms read as zero) in one
//      sum_gather launch per side -- a full, unclipped single +1 term is passed
//      through as a view instead;
//   2. M_r := S^A_r S^B_r by the level-2 program (into zeroed temporaries, with
//      alpha = 1 as AB / Naive do, variants.cpp:161);
//   3. one stream pass C_q += (alpha gamma) M_r in table order (variants.cpp:99-109).
// The products are those of the composed level-3 table (entry 49 r + inner);
// only the association of the operand-sum and update additions differs.
long run_outer(Engine& e, cudaStream_t s, strassen_variant variant, int level, double alpha,
               const DView& A, const DView& B, const DView& C) {
    const long m = A.rows, k = A.cols, n = B.cols;
    const long qm = ceil_div(m, 2), qk = ceil_div(k, 2), qn = ceil_div(n, 2);
    long launches = 0;
    const TmaOperand ta = prepare(e, s, A, qm, qk, 2, e.pack_a3, launches);
    const TmaOperand tb = prepare(e, s, B, qk, qn, 2, e.pack_b3, launches);
    std::vector<bool> a_live(4), b_live(4), c_live(4);
    std::vector<QuadView> cq(4);
    for (int I = 0; I < 2; ++I)
        for (int J = 0; J < 2; ++J) {
            a_live[I * 2 + J] = quad_rows(ta, I) > 0 && quad_cols(ta, J) > 0;
            b_live[I * 2 + J] = quad_rows(tb, I) > 0 && quad_cols(tb, J) > 0;
            cq[I * 2 + J] = c_quad(C, qm, qn, I, J);
            c_live[I * 2 + J] = cq[I * 2 + J].rows > 0 && cq[I * 2 + J].cols > 0;
        }
    struct Live {
        Terms a, b, c;
    };
    std::vector<Live> live;
    for (const Product& pr : program_for_level(1).products) {
        Live l{live_terms(pr.a, a_live), live_terms(pr.b, b_live), live_terms(pr.c, c_live)};
        if (l.a.empty() || l.b.empty() || l.c.empty()) continue;  // variants.cpp:131-133
        live.push_back(std::move(l));
    }
    if (live.empty()) return launches;

    // The outer program over a list of live products: their operand sums, products
    // and stream pass.  When the outer temporaries of all seven products would take
    // more than half the free device memory (the inner level-2 calls need the rest),
    // the products run in consecutive groups in table order -- the same operations
    // on every C element in the same order, so the same result.
    auto run_group = [&](const std::vector<Live>& live) {
        // outer operands: a view of the quadrant, or a materialised sum (ld multiple of 4)
        const long long lda_t = ((qm + 3) / 4) * 4, ldb_t = ((qk + 3) / 4) * 4;
        const long long ldm = ((qm + 3) / 4) * 4;
        std::vector<DView> opA(live.size()), opB(live.size());
        for (int sd = 0; sd < 2; ++sd) {
            const TmaOperand& t = sd == 0 ? ta : tb;
            const long rows = sd == 0 ? qm : qk, cols = sd == 0 ? qk : qn;
            const long long ld = sd == 0 ? lda_t : ldb_t;
            std::unique_ptr<SumBatchParams> SB(new SumBatchParams);
            std::memset(SB.get(), 0, sizeof(SumBatchParams));
            SB->rows = rows;
            SB->cols = cols;
            SB->ld = ld;
            std::vector<int> job_of(live.size(), -1);
            for (size_t p = 0; p < live.size(); ++p) {
                const Terms& terms = sd == 0 ? live[p].a : live[p].b;
                DView& op = sd == 0 ? opA[p] : opB[p];
                op.rows = rows;
                op.cols = cols;
                op.rs = 1;
                const int q0 = terms[0].first;
                if (terms.size() == 1 && terms[0].second == 1 && quad_rows(t, q0 / 2) == rows &&
                    quad_cols(t, q0 % 2) == cols) {
                    op.p = const_cast<double*>(quad_origin(t, q0 / 2, q0 % 2));
                    op.cs = t.ld;
                    op.ready = t.ready;
                    continue;
                }
                const int z = SB->njobs++;
                job_of[p] = z;
                SB->nterms[z] = static_cast<int>(terms.size());
                for (size_t u = 0; u < terms.size(); ++u) {
                    const int qi = terms[u].first;
                    SumTerm& st = SB->t[z][u];
                    st.x = quad_origin(t, qi / 2, qi % 2);
                    st.rows = static_cast<int>(quad_rows(t, qi / 2));
                    st.cols = static_cast<int>(quad_cols(t, qi % 2));
                    st.ld = t.ld;
                    st.coeff = terms[u].second;
                }
            }
            if (SB->njobs) {
                double* T = e.ensure(sd == 0 ? e.l3_a : e.l3_b,
                                     static_cast<size_t>(SB->njobs) * ld * cols * 8);
                for (size_t p = 0; p < live.size(); ++p) {
                    if (job_of[p] < 0) continue;
                    double* dst = T + static_cast<size_t>(job_of[p]) * ld * cols;
                    SB->dst[job_of[p]] = dst;
                    DView& op = sd == 0 ? opA[p] : opB[p];
                    op.p = dst;
                    op.cs = ld;
                }
                if (t.ready) ck(cudaStreamWaitEvent(s, t.ready, 0), "wait operand");
                e.prof_begin("sum_gather_kernel", s);
                ck(launch_sum_batch(*SB, s), sd == 0 ? "outer sums (A)" : "outer sums (B)");
                e.prof_end(s);
                ++launches;
            }
        }

        // products M_r = S^A_r S^B_r by the level-2 program, alpha = 1, into zeroed
        // temporaries (the inner stream pass / fused epilogue accumulates into M_r)
        const size_t mstride = static_cast<size_t>(ldm) * qn;
        double* M = e.ensure(e.l3_m, live.size() * mstride * 8);
        ck(cudaMemsetAsync(M, 0, live.size() * mstride * 8, s), "zero products");
        for (size_t p = 0; p < live.size(); ++p) {
            DView Mp;
            Mp.p = M + p * mstride;
            Mp.rows = qm;
            Mp.cols = qn;
            Mp.rs = 1;
            Mp.cs = ldm;
            launches += run_device(e, s, variant, level - 1, 1.0, opA[p], opB[p], Mp, nullptr);
        }

        // C_q += alpha gamma M_r, each quadrant's updates in table order
        std::unique_ptr<StreamParams> SP(new StreamParams);
        std::memset(SP.get(), 0, sizeof(StreamParams));
        for (int qi = 0; qi < 4; ++qi) {
            SP->cptr[qi] = cq[qi].p;
            SP->crows[qi] = static_cast<int>(cq[qi].rows);
            SP->ccols[qi] = static_cast<int>(cq[qi].cols);
        }
        for (size_t p = 0; p < live.size(); ++p)
            for (const auto& [q, coeff] : live[p].c) {
                SP->src_prod[q][SP->nsrc[q]] = static_cast<int8_t>(p);
                SP->src_coeff[q][SP->nsrc[q]] = static_cast<int8_t>(coeff);
                ++SP->nsrc[q];
            }
        bool vec = C.rs == 1 && C.cs % 2 == 0 && (reinterpret_cast<uintptr_t>(C.p) % 16) == 0;
        for (int qi = 0; qi < 4 && vec; ++qi) vec = (reinterpret_cast<uintptr_t>(cq[qi].p) % 16) == 0;
        SP->c_vec = vec ? 1 : 0;
        SP->rs_c = C.rs;
        SP->cs_c = C.cs;
        SP->mbase = M;
        SP->mstride = static_cast<long long>(mstride);
        SP->ldm = ldm;
        SP->alpha = alpha;
        SP->nquad = 4;
        SP->qm = static_cast<int>(qm);
        SP->qn = static_cast<int>(qn);
        SP->ksplit = 1;
        SP->r0 = 0;
        SP->r1 = static_cast<int>(qm);
        SP->c0 = 0;
        SP->c1 = static_cast<int>(qn);
        wait_ready(s, C);
        e.prof_begin("stream_gather_kernel", s);
        ck(launch_stream_update(*SP, s), "outer stream_update");
        e.prof_end(s);
        ++launches;
    };
    const double per_prod = 8.0 * (static_cast<double>(((qm + 3) / 4) * 4) * qk +
                                   static_cast<double>(((qk + 3) / 4) * 4) * qn +
                                   static_cast<double>(((qm + 3) / 4) * 4) * qn);
    // one shot when the new allocations it needs (beyond the outer buffers the ctx
    // already holds) take at most half the free memory
    double ja = 0.0, jb = 0.0;  // materialised outer sums (multi-term sides)
    for (const Live& l : live) {
        ja += l.a.size() > 1;
        jb += l.b.size() > 1;
    }
    const double np = static_cast<double>(live.size());
    const double side_a = 8.0 * static_cast<double>(((qm + 3) / 4) * 4) * qk;
    const double side_b = 8.0 * static_cast<double>(((qk + 3) / 4) * 4) * qn;
    const double side_m = 8.0 * static_cast<double>(((qm + 3) / 4) * 4) * qn;
    const double extra = std::max(0.0, ja * side_a - static_cast<double>(e.l3_a.bytes)) +
                         std::max(0.0, jb * side_b - static_cast<double>(e.l3_b.bytes)) +
                         std::max(0.0, np * side_m - static_cast<double>(e.l3_m.bytes));
    if (extra <= 0.0 || extra <= 0.5 * device_bytes_free()) {
        run_group(live);
        return launches;
    }
    if (e.capturing)
        throw Error(STRASSEN_ERR_ALLOC, "stream capture: the call's temporaries do not fit "
                                        "beside the ctx's workspace (product groups release it)");
    ck(cudaDeviceSynchronize(), "sync before releasing temporaries");
    for (DeviceBuffer* b : {&e.l3_a, &e.l3_b, &e.l3_m})
        if (b->ptr) {
            cudaFree(b->ptr);
            b->ptr = nullptr;
            b->bytes = 0;
        }
    const size_t g = std::max<size_t>(1, static_cast<size_t>(0.5 * device_bytes_free() / per_prod));
    for (size_t i0 = 0; i0 < live.size(); i0 += g) {
        const size_t i1 = std::min(live.size(), i0 + g);
        run_group(std::vector<Live>(live.begin() + static_cast<long>(i0),
                                    live.begin() + static_cast<long>(i1)));
    }
    return launches;
}
}  // namespace

long scale_device(Engine& e, cudaStream_t s, const DView& C, double beta) {
    (void)e;
    wait_ready(s, C);
    ck(launch_scale(C.p, C.rows, C.cols, C.rs, C.cs, beta, s), "scale");
    return 1;
}

}  // namespace sb200
