// Native SUMMA over the drop-in library (include/strassen_dist.h).
//
// The paper's distributed experiment is SUMMA with the local
// one/two-level Strassen as the rank-b update; the reference stops at the
// in-process rank-b schedule of its bench library (tools/bench_lib.cpp:56-71).
// This file is that experiment for a C caller: one handle per GPU, broadcasts
// along process rows and columns (NCCL resolved with dlopen, or a caller's
// transport), double-buffered panels on a communication stream, and
// strassen_gemm_device as the local update.  It uses only the public C ABI of
// the library plus the CUDA runtime.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "engine.hpp"
#include "strassen_dist.h"

namespace sb200 {
void set_last_error(const std::string& what);  // capi.cpp
}

namespace {

using sb200::Error;

// ------------------------------------------------------------------- schedule
void grid_for(int p, int& pr, int& pc) {
    if (p < 1) throw std::invalid_argument("dist: nranks must be >= 1");
    pr = 1;
    for (int r = 1; static_cast<long>(r) * r <= p; ++r)
        if (p % r == 0) pr = r;
    pc = p / pr;
}

// [g0, g0 + width) cut at multiples of per_owner.
std::vector<strassen_dist_piece> cut(long g0, long width, long per_owner) {
    std::vector<strassen_dist_piece> out;
    for (long g = g0; g < g0 + width;) {
        const long owner = g / per_owner, off = g % per_owner;
        const long w = std::min(per_owner - off, g0 + width - g);
        out.push_back({static_cast<int>(owner), off, w, g - g0});
        g += w;
    }
    return out;
}

void check_layout(long k, int pr, int pc, long b) {
    if (pr < 1 || pc < 1) throw std::invalid_argument("dist: grid must be at least 1 x 1");
    if (k < 1 || k % pr || k % pc) throw std::invalid_argument("dist: k must divide the grid");
    if (b < 1 || k % b) throw std::invalid_argument("dist: the panel width must divide k");
}

// ----------------------------------------------------------------------- NCCL
// Only the handful of entry points the schedule needs, resolved at run time so
// the library has no link-time dependency on NCCL.
struct Nccl {
    typedef struct { char internal[STRASSEN_DIST_ID_BYTES]; } UniqueId;
    typedef void* Comm;
    static constexpr int kFloat64 = 8;  // ncclFloat64 (nccl.h ncclDataType_t)
    int (*GetUniqueId)(UniqueId*) = nullptr;
    int (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
    int (*CommSplit)(Comm, int, int, Comm*, void*) = nullptr;
    int (*CommDestroy)(Comm) = nullptr;
    int (*CommCount)(Comm, int*) = nullptr;
    int (*CommUserRank)(Comm, int*) = nullptr;
    int (*Broadcast)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    void* lib = nullptr;

    static Nccl& get() {
        static Nccl n;
        static std::once_flag once;
        std::call_once(once, [] {
            for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
                n.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
                if (n.lib) break;
            }
            if (!n.lib) return;
            auto sym = [&](const char* s) { return dlsym(n.lib, s); };
            n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
            n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
            n.CommSplit = reinterpret_cast<decltype(n.CommSplit)>(sym("ncclCommSplit"));
            n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
            n.CommCount = reinterpret_cast<decltype(n.CommCount)>(sym("ncclCommCount"));
            n.CommUserRank = reinterpret_cast<decltype(n.CommUserRank)>(sym("ncclCommUserRank"));
            n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
            n.GetErrorString =
                reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
        });
        if (!n.lib || !n.GetUniqueId || !n.CommInitRank || !n.CommSplit || !n.CommDestroy ||
            !n.CommCount || !n.CommUserRank || !n.Broadcast)
            throw Error(STRASSEN_ERR_DEVICE, "dist: NCCL (libnccl.so.2) could not be loaded");
        return n;
    }
    void ck(int r, const char* what) const {
        if (r != 0)
            throw Error(STRASSEN_ERR_DEVICE, std::string(what) + ": " +
                                                 (GetErrorString ? GetErrorString(r) : "NCCL error"));
    }
};

struct NcclTransport {
    Nccl::Comm world = nullptr, row = nullptr, col = nullptr;
    bool own_world = false;
};

int nccl_bcast(void* user, int axis, const double* send, double* recv, size_t count, int root,
               void* stream) {
    auto* t = static_cast<NcclTransport*>(user);
    return Nccl::get().Broadcast(send, recv, count, Nccl::kFloat64, root, axis == 0 ? t->row : t->col,
                                 static_cast<cudaStream_t>(stream));
}

void nccl_destroy(void* user) {
    auto* t = static_cast<NcclTransport*>(user);
    try {
        Nccl& n = Nccl::get();
        if (t->row) n.CommDestroy(t->row);
        if (t->col) n.CommDestroy(t->col);
        if (t->world && t->own_world) n.CommDestroy(t->world);
    } catch (...) {
    }
    delete t;
}

void cu(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) throw Error(STRASSEN_ERR_ALLOC, what);
    if (e != cudaSuccess)
        throw Error(STRASSEN_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}

struct Buf {
    double* p = nullptr;
    size_t count = 0;
    void ensure(size_t n) {  // grow-only, like the ctx workspace
        if (n <= count) return;
        if (p) {
            cu(cudaDeviceSynchronize(), "dist: sync before growing a panel buffer");
            cudaFree(p);
            p = nullptr;
            count = 0;
        }
        cu(cudaMalloc(reinterpret_cast<void**>(&p), n * sizeof(double)), "dist: panel buffer");
        count = n;
    }
    ~Buf() {
        if (p) cudaFree(p);
    }
};

template <typename F>
strassen_status guarded(F&& f) {
    try {
        f();
        return STRASSEN_OK;
    } catch (const Error& e) {
        sb200::set_last_error(e.what());
        return e.status;
    } catch (const std::invalid_argument& e) {
        sb200::set_last_error(e.what());
        return STRASSEN_ERR_PARAM;
    } catch (const std::bad_alloc& e) {
        sb200::set_last_error(e.what());
        return STRASSEN_ERR_ALLOC;
    } catch (const std::exception& e) {
        sb200::set_last_error(e.what());
        return STRASSEN_ERR_PARAM;
    }
}

}  // namespace

// --------------------------------------------------------------------- mailbox
struct strassen_dist_mailbox {
    bool replay = false;
    // (axis, group index, sequence number inside the call) -> payload
    std::map<std::tuple<int, int, long>, std::pair<double*, size_t>> slots;
    ~strassen_dist_mailbox() {
        for (auto& kv : slots)
            if (kv.second.first) cudaFree(kv.second.first);
    }
};

// ---------------------------------------------------------------------- handle
struct strassen_dist {
    strassen_ctx* ctx = nullptr;
    strassen_dist_transport transport{};
    int rank = 0, pr = 1, pc = 1, row = 0, col = 0;
    int device = -1;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t start = nullptr, ready[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
    Buf abuf[2], bbuf[2], bstage;
    long last_launches = 0, last_panels = 0;
    // loopback transport state
    strassen_dist_mailbox* mailbox = nullptr;
    long seq[2] = {0, 0};

    ~strassen_dist() {
        if (transport.destroy) transport.destroy(transport.user);
        if (comm_stream) cudaStreamDestroy(comm_stream);
        for (cudaEvent_t e : {start, ready[0], ready[1], freed[0], freed[1]})
            if (e) cudaEventDestroy(e);
    }
};

namespace {

int mailbox_bcast(void* user, int axis, const double* send, double* recv, size_t count, int root,
                  void* stream) {
    auto* d = static_cast<strassen_dist*>(user);
    strassen_dist_mailbox* mb = d->mailbox;
    auto s = static_cast<cudaStream_t>(stream);
    const int group = axis == 0 ? d->row : d->col;
    const int me = axis == 0 ? d->col : d->row;
    const auto key = std::make_tuple(axis, group, d->seq[axis]++);
    if (!mb->replay) {
        if (me != root) return 0;  // receivers get nothing in the record pass
        auto& slot = mb->slots[key];
        if (slot.second < count) {
            if (slot.first) {
                if (cudaDeviceSynchronize() != cudaSuccess) return 1;
                cudaFree(slot.first);
            }
            slot = {nullptr, 0};
            if (cudaMalloc(reinterpret_cast<void**>(&slot.first), count * 8) != cudaSuccess) return 1;
            slot.second = count;
        }
        if (cudaMemcpyAsync(slot.first, send, count * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return 1;
        if (recv != send &&
            cudaMemcpyAsync(recv, send, count * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return 1;
        return 0;
    }
    auto it = mb->slots.find(key);
    if (it == mb->slots.end() || it->second.second < count) return 1;
    return cudaMemcpyAsync(recv, it->second.first, count * 8, cudaMemcpyDeviceToDevice, s) ==
                   cudaSuccess
               ? 0
               : 1;
}

strassen_dist* make_handle(strassen_ctx* ctx, const strassen_dist_transport& tr, int rank, int pr,
                           int pc) {
    if (pr < 1 || pc < 1) throw std::invalid_argument("dist: grid must be at least 1 x 1");
    if (rank < 0 || rank >= pr * pc) throw std::invalid_argument("dist: rank outside the grid");
    auto d = std::make_unique<strassen_dist>();
    d->ctx = ctx;
    d->rank = rank;
    d->pr = pr;
    d->pc = pc;
    d->row = rank / pc;
    d->col = rank % pc;
    cu(cudaGetDevice(&d->device), "dist: no CUDA device");
    cu(cudaStreamCreateWithFlags(&d->comm_stream, cudaStreamNonBlocking), "dist: comm stream");
    for (cudaEvent_t* e : {&d->start, &d->ready[0], &d->ready[1], &d->freed[0], &d->freed[1]})
        cu(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "dist: event");
    d->transport = tr;  // owned from here on
    return d.release();
}

// Column block copy (rows x cols doubles) between column-major buffers.
void copy2d(double* dst, long ldd, const double* src, long lds, long rows, long cols,
            cudaStream_t s) {
    cu(cudaMemcpy2DAsync(dst, static_cast<size_t>(ldd) * 8, src, static_cast<size_t>(lds) * 8,
                         static_cast<size_t>(rows) * 8, static_cast<size_t>(cols),
                         cudaMemcpyDeviceToDevice, s),
       "dist: panel copy");
}

struct Call {
    strassen_dist* d;
    long m_l, n_l, k_c, k_r, b, panels;
    const double* a;
    long lda;
    const double* bm;
    long ldb;
};

// Issues panel p's exchange step into buffer p % 2 on the communication stream.
void post(const Call& c, long p) {
    strassen_dist* d = c.d;
    const int s = static_cast<int>(p % 2);
    cudaStream_t cs = d->comm_stream;
    if (p >= 2) cu(cudaStreamWaitEvent(cs, d->freed[s], 0), "dist: wait for a free panel buffer");
    auto bcast = [&](int axis, const double* send, double* recv, size_t count, int root) {
        if (d->transport.bcast(d->transport.user, axis, send, recv, count, root, cs) != 0)
            throw Error(STRASSEN_ERR_DEVICE, "dist: broadcast failed");
    };
    // A panel (m_l x b, ld m_l): column pieces are contiguous in the buffer.
    double* ab = d->abuf[s].p;
    for (const strassen_dist_piece& pc : cut(p * c.b, c.b, c.k_c)) {
        double* dst = ab + pc.panel_off * c.m_l;
        const bool mine = d->col == pc.owner;
        const double* src = mine ? c.a + pc.local_off * c.lda : nullptr;
        if (d->pc == 1) {  // no process row to talk to
            copy2d(dst, c.m_l, src, c.lda, c.m_l, pc.width, cs);
            continue;
        }
        const double* send = dst;
        if (mine) {
            if (c.lda == c.m_l)
                send = src;  // the owner's columns are contiguous: broadcast them in place
            else
                copy2d(dst, c.m_l, src, c.lda, c.m_l, pc.width, cs);
        }
        bcast(0, send, dst, static_cast<size_t>(c.m_l) * pc.width, pc.owner);
    }
    // B panel (b x n_l, ld b): a row piece of width b fills the buffer; narrower
    // pieces arrive in contiguous staging (w x n_l) and are placed afterwards.
    double* bb = d->bbuf[s].p;
    const auto pieces = cut(p * c.b, c.b, c.k_r);
    for (const strassen_dist_piece& pc : pieces) {
        const bool mine = d->row == pc.owner;
        const double* src = mine ? c.bm + pc.local_off : nullptr;
        if (d->pr == 1) {
            copy2d(bb + pc.panel_off, c.b, src, c.ldb, pc.width, c.n_l, cs);
            continue;
        }
        const bool whole = pieces.size() == 1;
        double* dst = whole ? bb : d->bstage.p;
        const double* send = dst;
        if (mine) {
            if (whole && c.ldb == c.b)
                send = src;  // the owner's block is exactly the panel
            else
                copy2d(dst, pc.width, src, c.ldb, pc.width, c.n_l, cs);
        }
        bcast(1, send, dst, static_cast<size_t>(pc.width) * c.n_l, pc.owner);
        if (!whole) copy2d(bb + pc.panel_off, c.b, dst, pc.width, pc.width, c.n_l, cs);
    }
    cu(cudaEventRecord(d->ready[s], cs), "dist: panel ready");
}

struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess)
            prev = cur;
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

extern "C" {

strassen_status strassen_dist_grid(int nranks, int* pr_out, int* pc_out) {
    if (!pr_out || !pc_out) return STRASSEN_ERR_NULL;
    return guarded([&] { grid_for(nranks, *pr_out, *pc_out); });
}

long strassen_dist_default_panel(long k) {
    long b = k;
    while (b > 8192 && b % 2 == 0) b /= 2;
    return b;
}

strassen_status strassen_dist_panel_pieces(long k, int pr, int pc, long b, long p, int side,
                                           strassen_dist_piece* out, long cap, long* count_out) {
    if (!count_out || (!out && cap > 0)) return STRASSEN_ERR_NULL;
    return guarded([&] {
        check_layout(k, pr, pc, b);
        if (side != 0 && side != 1) throw std::invalid_argument("dist: side must be 0 (A) or 1 (B)");
        if (p < 0 || p >= k / b) throw std::invalid_argument("dist: panel index out of range");
        const auto pieces = cut(p * b, b, side == 0 ? k / pc : k / pr);
        *count_out = static_cast<long>(pieces.size());
        for (long t = 0; t < cap && t < *count_out; ++t) out[t] = pieces[t];
    });
}

strassen_status strassen_dist_unique_id(void* id_out) {
    if (!id_out) return STRASSEN_ERR_NULL;
    return guarded([&] {
        Nccl& n = Nccl::get();
        Nccl::UniqueId id;
        n.ck(n.GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id_out, &id, sizeof id);
    });
}

static strassen_status create_nccl(strassen_dist** out, strassen_ctx* ctx, Nccl::Comm world,
                                   bool own_world, int pr, int pc) {
    return guarded([&] {
        Nccl& n = Nccl::get();
        auto* t = new NcclTransport;
        t->world = world;
        t->own_world = own_world;
        strassen_dist_transport tr{nccl_bcast, nccl_destroy, t};
        try {
            int nranks = 0, rank = 0;
            n.ck(n.CommCount(world, &nranks), "ncclCommCount");
            n.ck(n.CommUserRank(world, &rank), "ncclCommUserRank");
            if (pr < 1 || pc < 1 || nranks != pr * pc)
                throw std::invalid_argument("dist: the communicator's size must equal pr * pc");
            // row communicator: the ranks of grid row i, ordered by column (root = column);
            // column communicator: the ranks of grid column j, ordered by row.
            n.ck(n.CommSplit(world, rank / pc, rank % pc, &t->row, nullptr), "ncclCommSplit(row)");
            n.ck(n.CommSplit(world, rank % pc, rank / pc, &t->col, nullptr), "ncclCommSplit(col)");
            *out = make_handle(ctx, tr, rank, pr, pc);
        } catch (...) {
            nccl_destroy(t);
            throw;
        }
    });
}

strassen_status strassen_dist_create(strassen_dist** out, strassen_ctx* ctx, const void* id,
                                     int rank, int nranks, int pr, int pc) {
    if (!out || !ctx || !id) return STRASSEN_ERR_NULL;
    *out = nullptr;
    Nccl::Comm world = nullptr;
    strassen_status st = guarded([&] {
        if (pr < 1 || pc < 1 || nranks != pr * pc)
            throw std::invalid_argument("dist: nranks must equal pr * pc");
        if (rank < 0 || rank >= nranks) throw std::invalid_argument("dist: rank outside the grid");
        Nccl& n = Nccl::get();
        Nccl::UniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        n.ck(n.CommInitRank(&world, nranks, uid, rank), "ncclCommInitRank");
    });
    if (st != STRASSEN_OK) return st;
    return create_nccl(out, ctx, world, true, pr, pc);
}

strassen_status strassen_dist_create_from_comm(strassen_dist** out, strassen_ctx* ctx,
                                               void* nccl_comm, int pr, int pc) {
    if (!out || !ctx || !nccl_comm) return STRASSEN_ERR_NULL;
    *out = nullptr;
    return create_nccl(out, ctx, nccl_comm, false, pr, pc);
}

strassen_status strassen_dist_create_custom(strassen_dist** out, strassen_ctx* ctx,
                                            const strassen_dist_transport* transport, int rank,
                                            int pr, int pc) {
    if (!out || !ctx || !transport || !transport->bcast) return STRASSEN_ERR_NULL;
    *out = nullptr;
    return guarded([&] {
        // the transport is owned only once the handle exists
        strassen_dist_transport borrowed = *transport;
        borrowed.destroy = nullptr;
        strassen_dist* d = make_handle(ctx, borrowed, rank, pr, pc);
        d->transport.destroy = transport->destroy;
        *out = d;
    });
}

strassen_status strassen_dist_mailbox_create(strassen_dist_mailbox** out) {
    if (!out) return STRASSEN_ERR_NULL;
    return guarded([&] { *out = new strassen_dist_mailbox; });
}

void strassen_dist_mailbox_destroy(strassen_dist_mailbox* mb) { delete mb; }

strassen_status strassen_dist_mailbox_set_replay(strassen_dist_mailbox* mb, int replay) {
    if (!mb) return STRASSEN_ERR_NULL;
    mb->replay = replay != 0;
    return STRASSEN_OK;
}

strassen_status strassen_dist_create_loopback(strassen_dist** out, strassen_ctx* ctx,
                                              strassen_dist_mailbox* mb, int rank, int pr, int pc) {
    if (!out || !ctx || !mb) return STRASSEN_ERR_NULL;
    *out = nullptr;
    return guarded([&] {
        strassen_dist* d = make_handle(ctx, strassen_dist_transport{mailbox_bcast, nullptr, nullptr},
                                       rank, pr, pc);
        d->transport.user = d;
        d->mailbox = mb;
        *out = d;
    });
}

void strassen_dist_destroy(strassen_dist* d) {
    if (!d) return;
    DeviceScope scope(d->device);
    cudaDeviceSynchronize();
    delete d;
}

strassen_status strassen_dist_gemm(strassen_dist* d, void* stream, strassen_variant variant,
                                   int level, long m, long n, long k, double alpha,
                                   const double* a, long lda, const double* b, long ldb,
                                   double* c, long ldc, long panel) {
    if (!d || !a || !b || !c) return STRASSEN_ERR_NULL;
    strassen_status inner = STRASSEN_OK;
    strassen_status st = guarded([&] {
        if (m < 1 || n < 1 || k < 1) throw std::invalid_argument("dist: dimensions must be >= 1");
        if (m % d->pr || n % d->pc) throw std::invalid_argument("dist: m, n must divide the grid");
        const long bw = panel > 0 ? panel : strassen_dist_default_panel(k);
        check_layout(k, d->pr, d->pc, bw);
        Call call{d, m / d->pr, n / d->pc, k / d->pc, k / d->pr, bw, k / bw, a, lda, b, ldb};
        if (lda < call.m_l || ldb < call.k_r || ldc < call.m_l)
            throw std::invalid_argument("dist: leading dimension below the block's rows");
        if (!sb200::is_device_pointer(a) || !sb200::is_device_pointer(b) ||
            !sb200::is_device_pointer(c))
            throw std::invalid_argument("dist: blocks must be device memory");
        DeviceScope scope(d->device);
        auto s = static_cast<cudaStream_t>(stream);
        const size_t acount = static_cast<size_t>(call.m_l) * bw;
        const size_t bcount = static_cast<size_t>(bw) * call.n_l;
        const int nbuf = call.panels > 1 ? 2 : 1;
        for (int t = 0; t < nbuf; ++t) {
            d->abuf[t].ensure(acount);
            d->bbuf[t].ensure(bcount);
        }
        // a B panel straddling process rows arrives piecewise in contiguous staging
        if (d->pr > 1 && call.k_r % bw) d->bstage.ensure(bcount);
        d->seq[0] = d->seq[1] = 0;
        d->last_launches = 0;
        d->last_panels = 0;
        // the blocks (and whatever produced them on `s`) come before the first exchange
        cu(cudaEventRecord(d->start, s), "dist: start event");
        cu(cudaStreamWaitEvent(d->comm_stream, d->start, 0), "dist: comm stream start");
        post(call, 0);
        for (long p = 0; p < call.panels; ++p) {
            if (p + 1 < call.panels) post(call, p + 1);
            const int sl = static_cast<int>(p % 2);
            cu(cudaStreamWaitEvent(s, d->ready[sl], 0), "dist: wait for the panel");
            inner = strassen_gemm_device(d->ctx, stream, variant, level, call.m_l, call.n_l, bw,
                                         alpha, d->abuf[sl].p, 1, call.m_l, d->bbuf[sl].p, 1, bw, c,
                                         1, ldc);
            if (inner != STRASSEN_OK) {
                // drain what was enqueued so the panel buffers are quiescent
                cudaStreamSynchronize(d->comm_stream);
                cudaStreamSynchronize(s);
                return;
            }
            long launches = 0;
            strassen_ctx_last_launches(d->ctx, &launches);
            d->last_launches += launches;
            d->last_panels += 1;
            cu(cudaEventRecord(d->freed[sl], s), "dist: buffer free event");
        }
    });
    return st != STRASSEN_OK ? st : inner;
}

strassen_status strassen_dist_last_counts(const strassen_dist* d, long* launches_out,
                                          long* panels_out) {
    if (!d) return STRASSEN_ERR_NULL;
    if (launches_out) *launches_out = d->last_launches;
    if (panels_out) *panels_out = d->last_panels;
    return STRASSEN_OK;
}

strassen_status strassen_dist_position(const strassen_dist* d, int* rank, int* pr, int* pc,
                                       int* row, int* col) {
    if (!d) return STRASSEN_ERR_NULL;
    if (rank) *rank = d->rank;
    if (pr) *pr = d->pr;
    if (pc) *pc = d->pc;
    if (row) *row = d->row;
    if (col) *col = d->col;
    return STRASSEN_OK;
}

}  // extern "C"
