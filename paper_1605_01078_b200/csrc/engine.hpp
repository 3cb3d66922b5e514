// Host engine: the B200 re-layering of the reference's L3 (variants.cpp) and
// the parts of L1 (blocking.cpp) that stay on the host.  It partitions the
// operands into quadrant views (ceil rule, matrix.cpp:8-35), stages host
// operands to the device, normalises layouts TMA cannot read, builds the
// per-launch product program from the composed operand table, and launches
// the kernels of kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include <functional>
#include <stdexcept>
#include <string>
#include <vector>
#include <string>

#include "strassen.h"

namespace sb200 {

// Error carrying an ABI status (mirrors the reference's exception -> status
// translation, capi.cpp:22-44).
struct Error : std::runtime_error {
    strassen_status status;
    Error(strassen_status s, const std::string& what) : std::runtime_error(what), status(s) {}
};

struct DeviceBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
};

// Device-side state of one ctx (the B200 counterpart of Workspace,
// blocking.hpp:33-42): grow-only buffers reused across calls.
struct Engine {
    int device = -1;
    int num_sms = 0;
    bool initialised = false;
    cudaStream_t user_stream = nullptr;
    bool has_user_stream = false;
    DeviceBuffer stage_a, stage_b, stage_c;   // host-operand staging
    DeviceBuffer pack_a, pack_b;              // TMA layout normalisation
    DeviceBuffer mbuf, tabuf, tbbuf;          // AB / Naive temporaries
    DeviceBuffer ticket_buf;                  // ordered fused-epilogue tickets
    DeviceBuffer unit_ctr_buf;                // persistent launches' unit counters
    DeviceBuffer fringe_buf;                  // k-chunk partials of the peeled fringe updates
    int unit_ctr_next = 0;                    // next counter (reset per call)
    // recorded on the call stream at the end of every call; the next call's stream
    // waits on it first, so a call on another stream cannot overwrite workspace
    // (sums, partials, tickets) that kernels of the previous call still read
    cudaEvent_t ev_last = nullptr;
    bool ev_last_recorded = false;
    // level 3 (B200 extension, strassen_ctx_set_max_level): the outer level's
    // layout normalisation, materialised operands and products (run_outer)
    DeviceBuffer pack_a3, pack_b3, l3_a, l3_b, l3_m;
    // ABC / AB: operand sides of up to this many terms are summed in the mm kernel,
    // longer ones materialised by the sum pass (run_strassen; 4 = fully fused)
    int fuse_max_terms = 2;  // strassen_ctx_set_fused_terms
    int max_level = 2;  // strassen_ctx_set_max_level: 3 admits Naive / C at level 3
    // strassen_ctx_set_operand_events: events the next call's kernels wait on right
    // before first reading A / B / C (device operands), then cleared
    cudaEvent_t next_ready[3] = {nullptr, nullptr, nullptr};
    long last_launches = 0;
    bool peeling = true;  // dynamic peeling of odd fringes (strassen_ctx_set_peeling)
    // optional per-launch timing of the last call (strassen_ctx_enable_profiling)
    bool profiling = false;
    // the current call is being captured into a CUDA graph (capi.cpp gemm_impl): the
    // workspace may not grow (growing synchronises the device)
    bool capturing = false;
    struct Timed {
        const char* name;
        cudaEvent_t start, stop;
    };
    std::vector<Timed> timed;
    void prof_begin(const char* name, cudaStream_t s);
    void prof_end(cudaStream_t s);
    std::string last_profile();  // JSON list of {"kernel", "ms", "start_ms"}

    ~Engine();
    void init();
    cudaStream_t stream();
    // host-operand staging: copies run on their own stream, one event each
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_call = nullptr, ev_ready[3] = {nullptr, nullptr, nullptr};
    // column-window pipeline of host calls (ColumnWindows): results leave on
    // their own stream so they overlap the next window's transfers and kernels
    bool pipelining = true;  // strassen_ctx_set_pipelining
    cudaStream_t d2h_stream = nullptr;
    cudaEvent_t ev_d2h = nullptr;
    static constexpr int kMaxStrips = 16, kMaxWindows = kMaxStrips * kMaxStrips;
    cudaEvent_t ev_win_a[kMaxStrips] = {}, ev_win_b[kMaxStrips] = {};
    cudaEvent_t ev_win_c[kMaxWindows] = {}, ev_win_done[kMaxWindows] = {};
    // windows alternate between the call stream and aux_stream so that one
    // window's tail wave overlaps the next window's first
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_sum_a[kMaxStrips] = {}, ev_sum_b[kMaxStrips] = {};
    double* ensure(DeviceBuffer& b, size_t bytes);
    size_t workspace_bytes() const;
};

struct DView {  // a strided matrix view in device memory
    double* p = nullptr;
    long rows = 0, cols = 0;
    long long rs = 0, cs = 0;
    // set when the view is still being copied in (host operand on the copy
    // stream): kernels that read it wait on this event right before launch
    cudaEvent_t ready = nullptr;
};

// Make stream s wait until view v has landed (no-op for resident operands).
inline void wait_ready(cudaStream_t s, const DView& v) {
    if (v.ready) cudaStreamWaitEvent(s, v.ready, 0);
}

// Host-call pipeline: the output is cut into R x Cn windows of the quadrant
// partition -- window w = r*Cn + c is quadrant rows [r*qrows, (r+1)*qrows) and
// quadrant columns [c*qcols, (c+1)*qcols) of every quadrant.  A arrives in R
// row strips, B in Cn column strips, C in windows; each window's result leaves
// as soon as it is final.  Windows run in growing shells (max(r, c) = 0, 1,
// ...), so each shell needs one new A strip and one new B strip while its
// compute grows: transfers of later windows overlap the kernels of earlier
// ones.  Per element the
// arithmetic is exactly that of the unwindowed call (same partition, same
// launch modes, same k order).
struct Windows {
    int rows = 0, cols = 0;              // R x Cn windows (0: none)
    // strip boundaries in quadrant rows / columns (rows + 1, cols + 1 entries;
    // tile multiples except the last)
    std::vector<long> rb, cb;
    std::function<void(int)> issue_a;    // enqueue A row strip r, record a_ready[r]
    std::function<void(int)> issue_b;    // enqueue B column strip c, record b_ready[c]
    std::function<void(int)> issue_c;    // enqueue C window w, record c_ready[w]
    std::function<void(int)> issue_out;  // enqueue window w's copy-back after done[w]
    cudaEvent_t* a_ready = nullptr;
    cudaEvent_t* b_ready = nullptr;
    cudaEvent_t* c_ready = nullptr;
    cudaEvent_t* done = nullptr;         // recorded on s after window w's last kernel
    int count() const { return rows * cols; }
};

// Processing order of an R x Cn window grid (window ids r*Cn + c): shells of
// max(r, c) = s, each as (0..s-1, s) then (s, 0..s).
std::vector<int> window_order(int rows, int cols);

// Window grid worth pipelining a host call into (rows = cols = 0: none).
// row_windows: A can arrive in row strips (host, column-major).
void plan_windows(const Engine& e, strassen_variant variant, int level, long m, long n, long k,
                  bool row_windows, Windows& w);

// C := alpha A B + C on device views, enqueued on `s` (no synchronisation).
// variant/level already validated.  Returns the number of kernel launches.
// With `win`, the operands arrive through win->issue_* (their views carry no
// ready event) and every window is handed to win->issue_out.
long run_device(Engine& e, cudaStream_t s, strassen_variant variant, int level, double alpha,
                const DView& A, const DView& B, const DView& C, const Windows* win = nullptr);

// C := beta C on a device view.
long scale_device(Engine& e, cudaStream_t s, const DView& C, double beta);

// Pointer classification for host staging.
bool is_device_pointer(const void* p);

}  // namespace sb200
