// sm_100a kernels of the B200 Strassen DGEMM.
//
// mm_kernel is the fused ABC Strassen tile kernel (it also runs the classical
// DGEMM as a one-product program and the AB / Naive / C product stages).  It
// replaces the reference's whole L1+L0 engine:
//   pack_a_sum / pack_b_sum      (blocking.cpp:12-66)  -> TMA operand-term loads
//                                   into a shared-memory ring; each DMMA warp sums
//                                   the terms of exactly the fragments it
//                                   multiplies, in registers
//   microkernel / accumulate     (kernel.cpp:8-47)     -> DMMA (mma.sync m8n8k4 f64)
//                                   mainloop over 64x32 warp tiles
//   multi-destination update     (kernel.cpp:49-76)    -> epilogue adding
//                                   alpha*gamma*M into each C quadrant tile: TMA
//                                   tensor reduce-adds from a staged tile, or a
//                                   register read-modify-write
//   five-loop driver + OpenMP ic (blocking.cpp:82-131) -> the CTA grid: one CTA per
//                                   (tile, product[, k-chunk]) or persistent CTAs
//                                   walking those units; per-tile tickets apply
//                                   every C tile's updates in table order, so the
//                                   results are bitwise deterministic run to run.
// Why DMMA, and why the sums sit in the DMMA warps' own instruction stream:
// DESIGN.md section 3 (profiles/r01_fp64_peak.log: DMMA 37.1 TF/s vs DFMA 34.2;
// DADDs issued by other warps starve while DMMA saturates the FP64 pipe).
#include <atomic>
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace sb200 {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Predicated arrive: no branch, so the caller's instruction stream stays one
// basic block (ptxas can overlap the work on either side).
__device__ __forceinline__ void mbar_arrive_if(uint64_t* bar, bool pred) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %1, 0;\n"
        "@p mbarrier.arrive.shared::cta.b64 _, [%0];\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(static_cast<int>(pred))
        : "memory");
}

// Ticket handshake of the ordered fused epilogue (acquire / release at GPU scope).
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Tickets of the ordered epilogue (MMParams::tickets): one per C tile, holding the
// number of products whose updates that tile has received.
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int* tile_ticket(const MMParams& P, int tm, int tn) {
    return P.tickets + tm * P.ticket_ld + tn;
}
// Wait until tile (tm, tn) has received the updates of products 0 .. p-1 (one thread):
// relaxed polling, then one acquire fence.
__device__ __forceinline__ void wait_ticket(const MMParams& P, int p, int tm, int tn) {
    const int* t = tile_ticket(P, tm, tn);
    while (ld_relaxed_gpu(t) != p) __nanosleep(64);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// Hand the tile on to product p + 1 (one thread, after p's updates are visible).
__device__ __forceinline__ void release_ticket(const MMParams& P, int p, int tm, int tn) {
    st_release_gpu(tile_ticket(P, tm, tn), p + 1);
}

// ---- tensor memory as a parking place for accumulators (pair_mode) ------------
// Warp w reaches TMEM lanes 32 (w % 4) .. + 31; warps w and w + 4 share them.  Parking
// slot k (k < kParkSlots: the first products of a group) of warp w is columns
// [256 k + 128 (w / 4), + 128) of a 512-column allocation.  A thread's 64 doubles are
// 128 words, in 4 chunks of 32 words: chunk h holds acc[2h + (i / 8)][(i / 2) % 4][i % 2]
// for i < 16 (lo word, hi word) -- exactly the (h) grouping of the stage writes.
constexpr int kParkSlots = 2;
constexpr uint32_t kTmemCols = 512;
__device__ __forceinline__ uint32_t tmem_addr(uint32_t base, int warp, int h, int slot) {
    return base + ((32u * static_cast<uint32_t>(warp & 3)) << 16) +
           static_cast<uint32_t>(slot * 256 + (warp >> 2) * 128 + h * 32);
}
#define SB200_R32(r) r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], r[8], r[9], r[10], r[11], \
    r[12], r[13], r[14], r[15], r[16], r[17], r[18], r[19], r[20], r[21], r[22], r[23], r[24],  \
    r[25], r[26], r[27], r[28], r[29], r[30], r[31]
__device__ __forceinline__ void tmem_st32(uint32_t ta, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
        "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),
        "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),
        "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t ta, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
#undef SB200_R32
// Park this warp's accumulator tile (64 doubles per thread) in tensor memory.
__device__ __forceinline__ void tmem_park(uint32_t base, int warp, int slot,
                                          const double (&acc)[8][4][2]) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const double v = acc[2 * h + (i >> 3)][(i >> 1) & 3][i & 1];
            r[2 * i] = static_cast<uint32_t>(__double2loint(v));
            r[2 * i + 1] = static_cast<uint32_t>(__double2hiint(v));
        }
        tmem_st32(tmem_addr(base, warp, h, slot), r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// Chunk h (16 doubles) of a group's combined update ca M_slot0 + cc M_slot1 + cb M, in
// that order ((cb M + ca M0) + cc M1; coefficients in {-1, 0, 1}, so a destination of
// one product is exactly +-M with no rounding): v[i] for acc[2h + i / 8][(i / 2) % 4][i % 2].
__device__ __forceinline__ void group_values(uint32_t base, int warp, int h, int ca, int cc,
                                             int cb, const double (&acc)[8][4][2], double (&v)[16]) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = cb * acc[2 * h + (i >> 3)][(i >> 1) & 3][i & 1];
#pragma unroll
    for (int k = 0; k < kParkSlots; ++k) {
        const int c = k == 0 ? ca : cc;
        if (c == 0) continue;
        uint32_t t[32];
        tmem_ld32(tmem_addr(base, warp, h, k), t);
#pragma unroll
        for (int i = 0; i < 16; ++i)
            v[i] = fma(static_cast<double>(c),
                       __hiloint2double(static_cast<int>(t[2 * i + 1]), static_cast<int>(t[2 * i])),
                       v[i]);
    }
}

// Tensor reduce-add smem -> global through a tensor map (f64 add at L2,
// UTMAREDG.2D.ADD); coordinates {row, column} of the box origin.
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, int c0, int c1,
                                                  const void* ssrc) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group"
        " [%0, {%1, %2}], [%3];" ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
        "r"(smem_u32(ssrc))
        : "memory");
}

// Named barrier over the DMMA warps only (the producer warp has exited): 8 warps,
// or the narrow-tile launch's 4.
template <int CW = kConsumerWarps>
__device__ __forceinline__ void consumer_bar() {
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
}

// Consumer side of a ring slot hand-back.  The slot was read with generic-proxy
// LDS; the producer refills it with TMA (async proxy).  Every lane fences its
// reads against the async proxy before lane 0 arrives -- without it ptxas may
// issue the arrive while this k-step's last LDS are still in flight (it hoists
// the predicated arrive above the trailing DMMAs), and a refill can then race
// the read.
__device__ __forceinline__ void consumer_fence() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// D(8x8) += A(8x4) B(4x8), fp64, one DMMA.8 on sm_100a.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// ---- shared-memory operand layouts and the DMMA fragment mapping ---------
// A tile (128 m x 16 k): 8 TMA boxes of {16 m, 16 k} with the 128-byte
// swizzle; double (m, k) at byte (m/16)*2048 + k*128 + (((m%16)/2 ^ k%8) << 4)
// + (m%2)*8.
// B tile (16 k x 128 n): one TMA box {16 k, 128 n}, 128-byte swizzle; double
// (k, n) at byte n*128 + (((k/2) ^ n%8) << 4) + (k%2)*8.
// A 16-k stage is 4 DMMA substeps s; lane (g = lane/4, j = lane%4) feeds
// physical k = p(s, j) = 2j + (s%2) + 8(s/2) (A and B agree, so the sum over
// k is unchanged).  Lane group g supplies A rows 16h + 2g + {0,1} of the
// fragment pair (2h, 2h+1) with one 16-byte load and B column
// nperm(g) = ((g%2)<<2) | (g/2) of each 8-column group, which also permutes
// the accumulator columns the epilogue writes.  With these choices every
// fragment load is a conflict-free 16-byte LDS (4 wavefronts per warp).
__device__ __forceinline__ int nperm(int c) { return ((c & 1) << 2) | (c >> 1); }

struct Frags {
    double a[2][8];  // [substep in pair][m fragment]
    double b[2][4];  // [substep in pair][n fragment]
};

// Fragment addresses of substeps 2*sp and 2*sp+1 inside an A / B tile.
__device__ __forceinline__ const uint8_t* frag_a_ptr(const uint8_t* sA, int ss, int sp, int wm,
                                                     int g, int j) {
    const int k = 2 * j + ss + 8 * sp;
    return sA + (wm * 4) * 2048 + k * 128 + ((g ^ (k & 7)) << 4);
}
__device__ __forceinline__ const uint8_t* frag_b_ptr(const uint8_t* sB, int sp, int wn, int g,
                                                     int j) {
    return sB + (wn * 32 + nperm(g)) * 128 + (((j + 4 * sp) ^ nperm(g)) << 4);
}

// Operand term u of one side, loaded and added into the fragments:
// acc (+)= c_u * x, c_u = +-1 applied as a sign flip so each add is one DADD
// rounding exactly like the reference's pack_a_sum / pack_b_sum accumulation
// (blocking.cpp:24-28; terms in listed order, the first one copied).
// FIRST: plain load (the caller negates afterwards in the rare -1 case);
// otherwise acc = fma(c, x, acc) with c = +-1, which rounds exactly like
// acc + c*x (c*x is exact) and needs no separate negation.
template <bool FIRST>
__device__ __forceinline__ void frag_a_term(const uint8_t* sA, int sp, int wm, int g, int j,
                                            double c, Frags& f) {
#pragma unroll
    for (int ss = 0; ss < 2; ++ss) {
        const uint8_t* pa = frag_a_ptr(sA, ss, sp, wm, g, j);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const double2 v = *reinterpret_cast<const double2*>(pa + h * 2048);
            if (FIRST) {
                f.a[ss][2 * h] = v.x;
                f.a[ss][2 * h + 1] = v.y;
            } else {
                f.a[ss][2 * h] = fma(c, v.x, f.a[ss][2 * h]);
                f.a[ss][2 * h + 1] = fma(c, v.y, f.a[ss][2 * h + 1]);
            }
        }
    }
}
template <bool FIRST>
__device__ __forceinline__ void frag_b_term(const uint8_t* sB, int sp, int wn, int g, int j,
                                            double c, Frags& f) {
    const uint8_t* pb = frag_b_ptr(sB, sp, wn, g, j);
#pragma unroll
    for (int nf = 0; nf < 4; ++nf) {
        const double2 v = *reinterpret_cast<const double2*>(pb + nf * 8 * 128);
        if (FIRST) {
            f.b[0][nf] = v.x;
            f.b[1][nf] = v.y;
        } else {
            f.b[0][nf] = fma(c, v.x, f.b[0][nf]);
            f.b[1][nf] = fma(c, v.y, f.b[1][nf]);
        }
    }
}

__device__ __forceinline__ void dmma_substep(const Frags& f, int ss, double (&acc)[8][4][2]) {
#pragma unroll
    for (int mf = 0; mf < 8; ++mf)
#pragma unroll
        for (int nf = 0; nf < 4; ++nf)
            dmma(acc[mf][nf][0], acc[mf][nf][1], f.a[ss][mf], f.b[ss][nf]);
}

// ---- A-heavy layout: 4 (m) x 2 (n) warps of 32 x 64 -----------------------
// For products with more A terms than B terms each A element is summed by two
// warps instead of four (the 2 x 4 layout's A-heavy products cost 6.5-8% more than
// their B-heavy mirrors, profiles/r01_abc2_combo_costs.log).  Accumulator (mf, nf)
// of this layout (mf < 4, nf < 8) lives in acc[(8 mf + nf) / 4][(8 mf + nf) % 4],
// and relayout_to_2x4 moves the tile back to the 2 x 4 layout the epilogues expect.
struct Frags1 {
    double a[2][4];  // [substep in pair][m fragment]
    double b[2][8];  // [substep in pair][n fragment]
};
template <bool FIRST>
__device__ __forceinline__ void frag_a_term1(const uint8_t* sA, int sp, int wm1, int g, int j,
                                             double c, Frags1& f) {
#pragma unroll
    for (int ss = 0; ss < 2; ++ss) {
        const int k = 2 * j + ss + 8 * sp;
        const uint8_t* pa = sA + (wm1 * 2) * 2048 + k * 128 + ((g ^ (k & 7)) << 4);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double2 v = *reinterpret_cast<const double2*>(pa + h * 2048);
            if (FIRST) {
                f.a[ss][2 * h] = v.x;
                f.a[ss][2 * h + 1] = v.y;
            } else {
                f.a[ss][2 * h] = fma(c, v.x, f.a[ss][2 * h]);
                f.a[ss][2 * h + 1] = fma(c, v.y, f.a[ss][2 * h + 1]);
            }
        }
    }
}
template <bool FIRST>
__device__ __forceinline__ void frag_b_term1(const uint8_t* sB, int sp, int wn1, int g, int j,
                                             double c, Frags1& f) {
    const uint8_t* pb = sB + (wn1 * 64 + nperm(g)) * 128 + (((j + 4 * sp) ^ nperm(g)) << 4);
#pragma unroll
    for (int nf = 0; nf < 8; ++nf) {
        const double2 v = *reinterpret_cast<const double2*>(pb + nf * 8 * 128);
        if (FIRST) {
            f.b[0][nf] = v.x;
            f.b[1][nf] = v.y;
        } else {
            f.b[0][nf] = fma(c, v.x, f.b[0][nf]);
            f.b[1][nf] = fma(c, v.y, f.b[1][nf]);
        }
    }
}
__device__ __forceinline__ void dmma_substep1(const Frags1& f, int ss, double (&acc)[8][4][2]) {
#pragma unroll
    for (int mf = 0; mf < 4; ++mf)
#pragma unroll
        for (int nf = 0; nf < 8; ++nf)
            dmma(acc[(8 * mf + nf) >> 2][(8 * mf + nf) & 3][0],
                 acc[(8 * mf + nf) >> 2][(8 * mf + nf) & 3][1], f.a[ss][mf], f.b[ss][nf]);
}

// ---- half-k tiles (ProductDesc::half: products with 4 + 4 terms) ----------
// A (4,4) product needs 8 term tiles per 16-k step; with 16-k tiles the ring
// could prefetch only a fraction of the next step, exposing TMA latency.  Such
// products stream 8-k half tiles instead, two per 16 KB slot (term u at slot
// u/2, byte offset (u%2)*8 KB), so the ring holds 3.5 steps.
// A half tile (128 m x 8 k): 8 boxes {16 m, 8 k}, 128-byte swizzle: (m, k) at
// (m/16)*1024 + k*128 + (((m%16)/2 ^ k) << 4) + (m%2)*8.
// B half tile (8 k x 128 n): one box {8 k, 128 n}, 64-byte swizzle: (k, n) at
// n*64 + (((k/2) ^ (n/2)%4) << 4) + (k%2)*8.
// Lane (g, j) feeds k = 2j + ss in both (the same k order as the 16-k path:
// bitwise-identical sums), A rows as in the 16-k path, and B column g
// (identity column map; the epilogue uses the matching accumulator columns).
// Both are conflict-free: per quarter-warp, A chunks g ^ k are 8 distinct,
// B lanes cover the two 64-byte halves (n parity) x 4 chunks.
constexpr int kHalfBytes = kSlotBytes / 2;

template <bool FIRST>
__device__ __forceinline__ void frag_a_half(const uint8_t* sA, int wm, int g, int j, double c,
                                            Frags& f) {
#pragma unroll
    for (int ss = 0; ss < 2; ++ss) {
        const int k = 2 * j + ss;
        const uint8_t* pa = sA + (wm * 4) * 1024 + k * 128 + ((g ^ k) << 4);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const double2 v = *reinterpret_cast<const double2*>(pa + h * 1024);
            if (FIRST) {
                f.a[ss][2 * h] = v.x;
                f.a[ss][2 * h + 1] = v.y;
            } else {
                f.a[ss][2 * h] = fma(c, v.x, f.a[ss][2 * h]);
                f.a[ss][2 * h + 1] = fma(c, v.y, f.a[ss][2 * h + 1]);
            }
        }
    }
}
template <bool FIRST>
__device__ __forceinline__ void frag_b_half(const uint8_t* sB, int wn, int g, int j, double c,
                                            Frags& f) {
    const uint8_t* pb = sB + (wn * 32 + g) * 64 + ((j ^ ((g >> 1) & 3)) << 4);
#pragma unroll
    for (int nf = 0; nf < 4; ++nf) {
        const double2 v = *reinterpret_cast<const double2*>(pb + nf * 8 * 64);
        if (FIRST) {
            f.b[0][nf] = v.x;
            f.b[1][nf] = v.y;
        } else {
            f.b[0][nf] = fma(c, v.x, f.b[0][nf]);
            f.b[1][nf] = fma(c, v.y, f.b[1][nf]);
        }
    }
}

// Half tiles of one 8-k step: term u (A terms first) in slot slot0 + u/2.
template <int NT>
struct HalfStep {
    const uint8_t* t[NT];
    uint32_t slot0;
};

template <int NT, int RING>
__device__ __forceinline__ void half_acquire(const uint8_t* raw, uint64_t* raw_full,
                                             uint32_t& slot, uint32_t& phase, HalfStep<NT>& hs) {
    constexpr int kSlots = (NT + 1) / 2;
    hs.slot0 = slot;
#pragma unroll
    for (int v = 0; v < kSlots; ++v) {
        uint32_t sv = slot + v;
        const uint32_t pv = (sv >= RING) ? phase ^ 1 : phase;
        sv = (sv >= RING) ? sv - RING : sv;
        hs.t[2 * v] = raw + sv * kSlotBytes;
        if (2 * v + 1 < NT) hs.t[2 * v + 1] = raw + sv * kSlotBytes + kHalfBytes;
        mbar_wait(&raw_full[sv], pv);
    }
    slot += kSlots;
    if (slot >= RING) {
        slot -= RING;
        phase ^= 1;
    }
}

template <int NT, int RING>
__device__ __forceinline__ void half_release(uint64_t* raw_empty, const HalfStep<NT>& hs,
                                             int lane) {
    consumer_fence();
    __syncwarp();
    uint32_t s2 = hs.slot0;
#pragma unroll
    for (int v = 0; v < (NT + 1) / 2; ++v) {
        mbar_arrive_if(&raw_empty[s2], lane == 0);  // predicated: no branch
        s2 = (s2 + 1 == RING) ? 0 : s2 + 1;
    }
}

// Hand the N ring slots from slot0 on back to the producer (predicated arrive: no
// branch).  Called right after the k-step's LAST fragment loads, before the DMMAs that
// consume them, so the refill of these slots overlaps the step's second half; the
// fence orders this warp's LDS before the async-proxy (TMA) writes that follow.
template <int N, int RING>
__device__ __forceinline__ void release_slots(uint64_t* raw_empty, uint32_t slot0, int lane) {
    consumer_fence();
    __syncwarp();
    uint32_t s2 = slot0;
#pragma unroll
    for (int u = 0; u < N; ++u) {
        mbar_arrive_if(&raw_empty[s2], lane == 0);
        s2 = (s2 + 1 == RING) ? 0 : s2 + 1;
    }
}

// One product's k-loop over half tiles: two 8-k steps per 16-k tile (both
// waits first, then one straight-line block that returns the first step's
// slots as soon as it is done).  kt_lo / kt_hi count 16-k tiles.
template <int NA, int NB, int RING>
__device__ __forceinline__ void product_kloop_half(const uint8_t* raw, uint64_t* raw_full,
                                                   uint64_t* raw_empty, uint32_t& slot,
                                                   uint32_t& phase, int kt_lo, int kt_hi,
                                                   const ProductDesc& pd, int wm, int wn, int g,
                                                   int j, int lane, double (&acc)[8][4][2]) {
    double ca[NA], cb[NB];
#pragma unroll
    for (int u = 0; u < NA; ++u) ca[u] = static_cast<double>(pd.as[u]);
#pragma unroll
    for (int u = 0; u < NB; ++u) cb[u] = static_cast<double>(pd.bs[u]);
    for (int kt = kt_lo; kt < kt_hi; ++kt) {
        HalfStep<NA + NB> h[2];
        half_acquire<NA + NB, RING>(raw, raw_full, slot, phase, h[0]);
        half_acquire<NA + NB, RING>(raw, raw_full, slot, phase, h[1]);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            Frags f;
            frag_a_half<true>(h[e].t[0], wm, g, j, 1.0, f);
            frag_b_half<true>(h[e].t[NA], wn, g, j, 1.0, f);
#pragma unroll
            for (int u = 1; u < NA; ++u) frag_a_half<false>(h[e].t[u], wm, g, j, ca[u], f);
#pragma unroll
            for (int u = 1; u < NB; ++u) frag_b_half<false>(h[e].t[NA + u], wn, g, j, cb[u], f);
            dmma_substep(f, 0, acc);
            dmma_substep(f, 1, acc);
            half_release<NA + NB, RING>(raw_empty, h[e], lane);  // first half's slots back mid-tile
        }
    }
}

// One product's k-loop with compile-time term counts (NA, NB): no branches
// inside a k-step, so ptxas can overlap the operand loads and sums of the next
// substep pair with the DMMAs of the current one.  The host normalises every
// product so its first A and B terms have coefficient +1 (negating the other
// terms and the destination coefficients instead: exact, round-to-nearest is
// sign-symmetric), so the first term is a plain load.
template <int NA, int NB, int RING>
__device__ __forceinline__ void product_kloop(const uint8_t* raw, uint64_t* raw_full,
                                              uint64_t* raw_empty, uint32_t& slot,
                                              uint32_t& phase, int kt_lo, int kt_hi,
                                              const ProductDesc& pd, int wm, int wn, int g,
                                              int j, int lane, double (&acc)[8][4][2]) {
    double ca[NA], cb[NB];
#pragma unroll
    for (int u = 0; u < NA; ++u) ca[u] = static_cast<double>(pd.as[u]);
#pragma unroll
    for (int u = 0; u < NB; ++u) cb[u] = static_cast<double>(pd.bs[u]);
    for (int kt = kt_lo; kt < kt_hi; ++kt) {
        const uint8_t* sA[NA];
        const uint8_t* sB[NB];
        const uint32_t slot0 = slot;
#pragma unroll
        for (int u = 0; u < NA + NB; ++u) {
            uint32_t su = slot0 + u;
            const uint32_t pu = (su >= RING) ? phase ^ 1 : phase;
            su = (su >= RING) ? su - RING : su;
            if (u < NA) sA[u] = raw + su * kSlotBytes;
            else sB[u - NA] = raw + su * kSlotBytes;
            mbar_wait(&raw_full[su], pu);
        }
        slot += NA + NB;
        if (slot >= RING) {
            slot -= RING;
            phase ^= 1;
        }
#pragma unroll
        for (int sp = 0; sp < 2; ++sp) {
            Frags f;
            frag_a_term<true>(sA[0], sp, wm, g, j, 1.0, f);
            frag_b_term<true>(sB[0], sp, wn, g, j, 1.0, f);
#pragma unroll
            for (int u = 1; u < NA; ++u) frag_a_term<false>(sA[u], sp, wm, g, j, ca[u], f);
#pragma unroll
            for (int u = 1; u < NB; ++u) frag_b_term<false>(sB[u], sp, wn, g, j, cb[u], f);
            if (sp == 1) release_slots<NA + NB, RING>(raw_empty, slot0, lane);
            dmma_substep(f, 0, acc);
            dmma_substep(f, 1, acc);
        }
    }
}

// product_kloop in the 4 x 2 warp layout (A-heavy products, one CTA per unit).
template <int NA, int NB, int RING>
__device__ __forceinline__ void product_kloop1(const uint8_t* raw, uint64_t* raw_full,
                                               uint64_t* raw_empty, uint32_t& slot,
                                               uint32_t& phase, int kt_lo, int kt_hi,
                                               const ProductDesc& pd, int wm1, int wn1, int g,
                                               int j, int lane, double (&acc)[8][4][2]) {
    double ca[NA], cb[NB];
#pragma unroll
    for (int u = 0; u < NA; ++u) ca[u] = static_cast<double>(pd.as[u]);
#pragma unroll
    for (int u = 0; u < NB; ++u) cb[u] = static_cast<double>(pd.bs[u]);
    for (int kt = kt_lo; kt < kt_hi; ++kt) {
        const uint8_t* sA[NA];
        const uint8_t* sB[NB];
        const uint32_t slot0 = slot;
#pragma unroll
        for (int u = 0; u < NA + NB; ++u) {
            uint32_t su = slot0 + u;
            const uint32_t pu = (su >= RING) ? phase ^ 1 : phase;
            su = (su >= RING) ? su - RING : su;
            if (u < NA) sA[u] = raw + su * kSlotBytes;
            else sB[u - NA] = raw + su * kSlotBytes;
            mbar_wait(&raw_full[su], pu);
        }
        slot += NA + NB;
        if (slot >= RING) {
            slot -= RING;
            phase ^= 1;
        }
#pragma unroll
        for (int sp = 0; sp < 2; ++sp) {
            Frags1 f;
            frag_a_term1<true>(sA[0], sp, wm1, g, j, 1.0, f);
            frag_b_term1<true>(sB[0], sp, wn1, g, j, 1.0, f);
#pragma unroll
            for (int u = 1; u < NA; ++u) frag_a_term1<false>(sA[u], sp, wm1, g, j, ca[u], f);
#pragma unroll
            for (int u = 1; u < NB; ++u) frag_b_term1<false>(sB[u], sp, wn1, g, j, cb[u], f);
            if (sp == 1) release_slots<NA + NB, RING>(raw_empty, slot0, lane);
            dmma_substep1(f, 0, acc);
            dmma_substep1(f, 1, acc);
        }
    }
}

// The C tile from the 4 x 2 warp layout to the 2 x 4 one, through the (idle) ring:
// a 128 x 129-double row-major scratch (the pad spreads the banks).
__device__ __forceinline__ void relayout_to_2x4(uint8_t* raw, double (&acc)[8][4][2], int warp,
                                                int g, int j) {
    double* T = reinterpret_cast<double*>(raw);
    constexpr int LD = kBN + 1;
    const int c0 = nperm(2 * j), c1 = nperm(2 * j + 1);
    consumer_bar();  // every warp is done reading the ring
    {
        const int wm1 = warp & 3, wn1 = warp >> 2;
#pragma unroll
        for (int mf = 0; mf < 4; ++mf)
#pragma unroll
            for (int nf = 0; nf < 8; ++nf)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int row = wm1 * 32 + 16 * (mf >> 1) + 2 * g + (mf & 1);
                    const int col = wn1 * 64 + 8 * nf + (e ? c1 : c0);
                    T[row * LD + col] = acc[(8 * mf + nf) >> 2][(8 * mf + nf) & 3][e];
                }
    }
    consumer_bar();
    {
        const int wm = warp & 1, wn = warp >> 1;
#pragma unroll
        for (int mf = 0; mf < 8; ++mf)
#pragma unroll
            for (int nf = 0; nf < 4; ++nf)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int row = wm * 64 + 16 * (mf >> 1) + 2 * g + (mf & 1);
                    const int col = wn * 32 + 8 * nf + (e ? c1 : c0);
                    acc[mf][nf][e] = T[row * LD + col];
                }
    }
    consumer_bar();  // the ring is free for the epilogue's stage again
}

// One work unit of an mm launch: a C tile and the products / k-range it runs.
// piece / npieces: this unit's k-range is piece `piece` of the `npieces` that
// make up its (tile, product) -- k-chunks in split mode, stream-K pieces.
struct Unit {
    int tm, tn, p_lo, p_hi, kt_lo, kt_hi;
    int piece, npieces;
    int tk;  // ticket value of the unit's C update: its product, or its pair (pair_mode)
};
template <bool GROUPS>
__device__ __forceinline__ int unit_count(const MMParams& P) {
    if (P.streamk) return P.grid_cap * P.sk_maxp;
    if (GROUPS) return P.tiles_m * P.tiles_n * P.npairs;
    return P.tiles_m * P.tiles_n * (P.split ? P.nprod * P.ksplit : 1);
}
// unit -> (tile, product, k-chunk) in split mode, tile (all products) otherwise;
// tiles in grouped raster order (group_m tile rows share B column panels in L2)
template <bool GROUPS>
__device__ __forceinline__ Unit decode_unit(const MMParams& P, int bid) {
    Unit U;
    U.p_lo = 0;
    U.p_hi = P.nprod;
    U.kt_lo = 0;
    U.kt_hi = P.ktiles;
    U.piece = 0;
    U.npieces = 1;
    if (P.streamk) {
        // stream-K: CTA c covers k-steps [c*len, (c+1)*len) of the flattened
        // (product, tile, k-step) space (product-major); its j-th unit is its piece
        // of (tile, product) index tp0 + j (an empty unit when the range ends
        // earlier).  The pieces of index tp, in k order, come from CTAs
        // tp*K/len .. ((tp+1)*K-1)/len.
        const int grid = static_cast<int>(gridDim.x);
        const int c = bid % grid, jx = bid / grid;
        const long long K = P.ktiles, len = P.sk_len;
        const long long ntiles = static_cast<long long>(P.tiles_m) * P.tiles_n;
        const long long total = ntiles * P.nprod * K;
        const long long lo = c * len, hi = min(lo + len, total);
        const long long tp = lo / K + jx;
        const long long t_lo = tp * K;
        const bool live = lo < hi && t_lo < hi;
        U.p_lo = live ? static_cast<int>(tp / ntiles) : 0;
        U.p_hi = live ? U.p_lo + 1 : 0;  // empty unit: no product
        U.kt_lo = static_cast<int>(max(lo, t_lo) - t_lo);
        U.kt_hi = static_cast<int>(min(hi, t_lo + K) - t_lo);
        U.piece = c - static_cast<int>(t_lo / len);
        U.npieces = static_cast<int>((t_lo + K - 1) / len - t_lo / len + 1);
        bid = live ? static_cast<int>(tp % ntiles) : 0;
    } else if (P.split && P.unit_group > 0 && P.ksplit == 1) {
        // groups of G tiles, product-major inside: unit (t, p) of group g is
        // g*G*nprod + p*gt + t; the ticket a unit waits for, (t, p-1), always
        // has a smaller index (every earlier group is full)
        const int ntiles = P.tiles_m * P.tiles_n;
        const int G = P.unit_group;
        const int grp = bid / (G * P.nprod);
        const int rem = bid - grp * G * P.nprod;
        const int gt = min(G, ntiles - grp * G);
        U.p_lo = rem / gt;
        U.p_hi = U.p_lo + 1;
        bid = grp * G + rem % gt;
    } else if (GROUPS) {
        // (tile, group) units, group-major: the ticket a unit waits for, (t, j - 1), has
        // a smaller index
        const int ntiles = P.tiles_m * P.tiles_n;
        U.tk = bid / ntiles;
        U.p_lo = P.pair_lo[U.tk];
        U.p_hi = P.pair_lo[U.tk + 1];
        bid %= ntiles;
    } else if (P.split) {
        const int ntiles = P.tiles_m * P.tiles_n;
        const int s_idx = (bid / ntiles) % P.ksplit;
        U.p_lo = bid / (ntiles * P.ksplit);
        U.p_hi = U.p_lo + 1;
        U.kt_lo = s_idx * P.kt_per_split;
        U.kt_hi = min(P.ktiles, U.kt_lo + P.kt_per_split);
        U.piece = s_idx;
        U.npieces = P.ksplit;
        bid %= ntiles;
    }
    if (!GROUPS) U.tk = U.p_lo;
    const int per_group = P.group_m * P.tiles_n;
    const int grp = bid / per_group;
    const int first_m = grp * P.group_m;
    const int gsz = min(P.tiles_m - first_m, P.group_m);
    const int rr = bid - grp * per_group;
    U.tm = first_m + rr % gsz + P.tm0;
    U.tn = rr / gsz + P.tn0;
    return U;
}

// Cooperative fixup (MMParams::coop_fixup): the pieces of unit `bid`'s (tile, product)
// that finish it together -- this piece's index among them (-1: it only hands its
// partial over) and their number.  Stream-K: every piece that ends its CTA's range,
// i.e. all but a tail piece whose CTA goes on to the next (tile, product); k-chunk
// grids (one resident CTA per unit): every piece.  Computed after the mainloop (kept
// out of Unit: two more values live across the k-loop spill inside it).
__device__ __forceinline__ void coop_participants(const MMParams& P, int bid, int piece, int npieces,
                                               int& part, int& nparts) {
    part = piece;
    nparts = npieces;
    if (!P.streamk) return;
    const int grid = static_cast<int>(gridDim.x);
    const int c = bid % grid, jx = bid / grid;
    const long long K = P.ktiles, len = P.sk_len;
    const long long total = static_cast<long long>(P.tiles_m) * P.tiles_n * P.nprod * K;
    const long long t_lo = (c * len / K + jx) * K;
    const long long c_last = (t_lo + K - 1) / len;
    const bool tail_ends = min((c_last + 1) * len, total) == t_lo + K;
    nparts = npieces - (tail_ends ? 0 : 1);
    part = piece < nparts ? piece : -1;
}

// Cooperative fixup, run by a participant after its unit loop (it has stored its partial
// and arrived): wait for all the pieces of the tile, then finish the 64 x 8
// fragment blocks b = 4 warp + nf with b % nparts == part of its tile straight from the
// partials -- per element M = ((P_0 + P_1) + ...) + P_{n-1} in piece (k) order, the
// single-owner fixup's arithmetic -- and applies the epilogue to them: the C update of a
// one-product program, or the store of M_p.  mrow0 / ncol0 / c0 / c1: the lane's fragment
// origin and column pair, as in mm_kernel's epilogue.
template <int CW>
__device__ __forceinline__ void coop_finish(const MMParams& P, const ProductDesc& pd, int p, int tm,
                                            int tn, int mrow0, int ncol0, int c0, int c1, int warp,
                                            int part, int nparts, int npieces) {
    const long long ldm = P.ldm;
    int* cnt = P.arrive + (tm * P.ticket_ld + tn) * P.nprod + p;
    const double* Mq = P.mbase + P.part_off + static_cast<long long>(p * P.ksplit) * P.mstride;
    if (threadIdx.x == 0) {
        while (ld_relaxed_gpu(cnt) != npieces) __nanosleep(32);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    consumer_bar<CW>();
    // (a variant with both of a warp's blocks and their C values in flight together
    // measured slower: 768^3 DGEMM 45.0 -> 48.2 us)
    for (int nf = 0; nf < 4; ++nf) {
        if ((warp * 4 + nf) % nparts != part) continue;
        double2 v[4][2];
        // four pieces' loads in flight together, added in piece order
        for (int sp0 = 0; sp0 < npieces; sp0 += 4) {
            double2 x[4][4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double* Ms = Mq + static_cast<long long>(sp0 + i) * P.mstride;
#pragma unroll
                for (int h = 0; h < 4; ++h)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int row = mrow0 + 16 * h;
                        const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                        x[i][h][e] = make_double2(0.0, 0.0);
                        if (sp0 + i < npieces && col < P.qn && row < P.qm)
                            x[i][h][e] = __ldcg(reinterpret_cast<const double2*>(
                                Ms + row + static_cast<long long>(col) * ldm));
                    }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (sp0 + i >= npieces) break;
#pragma unroll
                for (int h = 0; h < 4; ++h)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        if (sp0 + i == 0) {
                            v[h][e] = x[i][h][e];
                        } else {
                            v[h][e].x += x[i][h][e].x;
                            v[h][e].y += x[i][h][e].y;
                        }
                    }
            }
        }
        // the block's epilogue: rows (2g, 2g + 1) + 16h, columns 8nf + c0 / c1
        if (P.mode == kEpiRMW) {
            for (int u = 0; u < pd.nc; ++u) {
                const int cq = pd.cq[u];
                double* __restrict__ C = P.cptr[cq];
                const int R = P.crows[cq], Cc = P.ccols[cq];
                const double sc = P.alpha * static_cast<double>(pd.cs[u]);
#pragma unroll
                for (int h = 0; h < 4; ++h)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int row = mrow0 + 16 * h;
                        const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                        if (col >= Cc) continue;
                        if (P.c_vec && row + 1 < R) {
                            double2* dst = reinterpret_cast<double2*>(
                                C + row + static_cast<long long>(col) * P.cs_c);
                            double2 cv = __ldcg(dst);
                            cv.x = fma(sc, v[h][e].x, cv.x);
                            cv.y = fma(sc, v[h][e].y, cv.y);
                            *dst = cv;
                        } else {
                            if (row < R) {
                                double* x0 = C + row * P.rs_c + static_cast<long long>(col) * P.cs_c;
                                *x0 = fma(sc, v[h][e].x, __ldcg(x0));
                            }
                            if (row + 1 < R) {
                                double* x1 = C + (row + 1) * P.rs_c + static_cast<long long>(col) * P.cs_c;
                                *x1 = fma(sc, v[h][e].y, __ldcg(x1));
                            }
                        }
                    }
            }
        } else {
            double* __restrict__ M = P.mbase + static_cast<long long>(p) * P.mstride;
#pragma unroll
            for (int h = 0; h < 4; ++h)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int row = mrow0 + 16 * h;
                    const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                    if (col >= P.qn) continue;
                    double* dst = M + row + static_cast<long long>(col) * ldm;
                    if (row + 1 < P.qm) {
                        asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(dst), "d"(v[h][e].x),
                                     "d"(v[h][e].y)
                                     : "memory");
                    } else if (row < P.qm) {
                        dst[0] = v[h][e].x;
                    }
                }
        }
    }
}

// Each CTA processes units blockIdx.x, + gridDim.x, ... in increasing order.
// With one CTA per unit that is a single pass; a persistent launch (one CTA
// per SM) keeps the producer streaming the next unit's operand tiles into the
// ring while the DMMA warps finish the current unit's epilogue.  Ticket waits
// only ever point at smaller units, which every CTA reaches first, so
// persistence cannot deadlock them.
//
// RING < kRawSlots (persistent single-term launches with short k): a smaller
// ring plus a separate bulk-reduction stage.  A CTA issues a unit's C
// reductions and goes straight on to the next unit's mainloop; the reductions'
// completion, and the ticket release that depends on it, are collected at the
// start of its next epilogue (or after its last unit).  A CTA always releases
// its deferred ticket before it waits on any ticket, so the ordering argument
// above still holds.
// Register form of the row-pair stream pass for the full level-1 / level-2 tables:
// the destination quadrants of every product are compile-time constants (the
// one-level table, table.cpp:18-33, composed as table.cpp:47-67 does -- in
// constexpr code here, so nothing is hand-entered twice), so the 4^L C
// accumulators live in registers instead of shared memory (the shared-memory
// form spends ~2 LDS/STS per update and was bound by them).  Per element the
// updates are the same fma's in the same order: bitwise identical results.
// The host uses it only when the call's (product -> destination quadrant) lists
// equal the table's.
struct StreamTab {
    int np;
    int nd[kMaxProducts];
    int dq[kMaxProducts][kMaxQuad];
};
constexpr StreamTab stream_tab_l1() {
    StreamTab t{};
    // C updates of M0..M6 (quadrant 2 * row + col), table.cpp:18-33
    const int d[7][2] = {{0, 3}, {2, 3}, {1, 3}, {0, 2}, {1, 0}, {3, -1}, {0, -1}};
    t.np = 7;
    for (int p = 0; p < 7; ++p) {
        t.nd[p] = d[p][1] < 0 ? 1 : 2;
        for (int u = 0; u < t.nd[p]; ++u) t.dq[p][u] = d[p][u];
    }
    return t;
}
constexpr StreamTab stream_tab_compose(const StreamTab& o, const StreamTab& in) {
    StreamTab t{};
    t.np = o.np * in.np;
    for (int a = 0; a < o.np; ++a)
        for (int b = 0; b < in.np; ++b) {
            const int p = a * in.np + b;
            t.nd[p] = 0;
            for (int u = 0; u < o.nd[a]; ++u)
                for (int v = 0; v < in.nd[b]; ++v) {
                    const int oq = o.dq[a][u], iq = in.dq[b][v];
                    const int row = 2 * (oq / 2) + iq / 2, col = 2 * (oq % 2) + iq % 2;
                    t.dq[p][t.nd[p]++] = row * 4 + col;
                }
        }
    return t;
}
// each product's destinations in ascending quadrant order, as the gather form lists
// them (to_gather below); per C element the update order is unchanged (ascending p)
constexpr StreamTab stream_tab_sorted(StreamTab t) {
    for (int p = 0; p < t.np; ++p)
        for (int a = 1; a < t.nd[p]; ++a)
            for (int b = a; b > 0 && t.dq[p][b - 1] > t.dq[p][b]; --b) {
                const int x = t.dq[p][b];
                t.dq[p][b] = t.dq[p][b - 1];
                t.dq[p][b - 1] = x;
            }
    return t;
}
constexpr StreamTab kStreamTab1 = stream_tab_sorted(stream_tab_l1());
constexpr StreamTab kStreamTab2 = stream_tab_sorted(stream_tab_compose(stream_tab_l1(), stream_tab_l1()));
template <int L>
__host__ __device__ constexpr const StreamTab& stream_tab() { return L == 1 ? kStreamTab1 : kStreamTab2; }

#ifdef SB200_TRACE
__device__ __forceinline__ void trace_event(const MMParams& P, int slot) {
    if (P.trace && threadIdx.x == 0 && slot < 32 && blockIdx.x < 8192) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.trace[blockIdx.x * 32 + slot] = t;
    }
}
#else
__device__ __forceinline__ void trace_event(const MMParams&, int) {}
#endif

// GROUPS: the launch runs product groups (MMParams::pair_mode); the other
// instantiations carry none of their tensor-memory and multi-coefficient epilogue code
template <int MAXT, bool PERSIST, int RING, bool GROUPS, bool NAR>
__global__ void __launch_bounds__(NAR ? kNarrowThreads : kThreads, NAR ? 2 : 1)
    mm_kernel(const __grid_constant__ MMParams P) {
    constexpr bool SEP = !NAR && RING != kRawSlots;  // separate stage, deferred completion
    // NAR: narrow tiles (kernels.hpp kNarrowBN): 4 DMMA warps, 64-column tiles
    constexpr int CW = NAR ? kNarrowConsumerWarps : kConsumerWarps;
    constexpr int BN = NAR ? kNarrowBN : kBN;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment (128B-swizzle atoms) by offsetting the shared array
    // itself, so every derived pointer stays in the shared address space (LDS/STS).
    uint8_t* raw = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* raw_full = reinterpret_cast<uint64_t*>(raw + RING * kSlotBytes);
    uint64_t* raw_empty = raw_full + RING;
    // dynamic unit hand-out (persistent launches): the TMA lane takes the next unit
    // from P.unit_counter and passes it to the DMMA warps through a small queue
    uint64_t* q_full = raw_empty + RING;
    uint64_t* q_empty = q_full + kUnitQueue;
    int* q_unit = reinterpret_cast<int*>(q_empty + kUnitQueue);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // cooperative fixup (MMParams::coop_fixup): the share of a (tile, product) this CTA
    // finishes after its unit loop -- {pending, p, tm, tn, part, nparts, npieces, half}
    __shared__ int coop_job[8];
    if (threadIdx.x == 0) coop_job[0] = 0;

    // PERSIST = false: exactly one unit per CTA (keeps the 4-term instantiation,
    // which runs at the register limit, free of the loop state)
    const int n_units = PERSIST ? unit_count<GROUPS>(P) : static_cast<int>(blockIdx.x) + 1;
    const bool persistent = PERSIST && static_cast<int>(gridDim.x) < n_units;
    const bool dyn = persistent && P.unit_counter != nullptr && !P.streamk;

    if (threadIdx.x == 0) {
        for (int s = 0; s < RING; ++s) {
            mbar_init(&raw_full[s], 1);
            mbar_init(&raw_empty[s], CW);
        }
        for (int s = 0; s < kUnitQueue; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
    }
    // GROUPS: warp 0 (a DMMA warp, which also frees it) allocates the tensor memory
    // the first products of a group are parked in
    uint32_t tmem_base = 0u;
    if constexpr (GROUPS) {
        __shared__ uint32_t tmem_base_s;
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(&tmem_base_s)),
                         "n"(kTmemCols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tmem_base = tmem_base_s;
    } else {
        __syncthreads();
    }
    // Unit sequence of this CTA: blockIdx.x first; then either a fixed stride of
    // gridDim.x, or (dyn) units taken from the global counter, in increasing order
    // across the grid.  The producer takes a unit when it starts streaming its tiles
    // and queues it for the DMMA warps, which take it when they finish the previous
    // one; an index >= n_units ends both loops.
    uint32_t qslot = 0, qphase = 0;
    auto producer_next = [&](int unit) -> int {
        if (!dyn) return unit + (PERSIST ? static_cast<int>(gridDim.x) : 1);
        const int nxt = static_cast<int>(gridDim.x) + atomicAdd(P.unit_counter, 1);
        mbar_wait(&q_empty[qslot], qphase ^ 1);
        *reinterpret_cast<volatile int*>(&q_unit[qslot]) = nxt;
        mbar_arrive(&q_full[qslot]);  // release: the DMMA warps' wait acquires the write
        if (++qslot == kUnitQueue) {
            qslot = 0;
            qphase ^= 1;
        }
        return nxt;
    };
    auto consumer_next = [&](int unit) -> int {
        if (!dyn) return unit + (PERSIST ? static_cast<int>(gridDim.x) : 1);
        mbar_wait(&q_full[qslot], qphase);
        const int nxt = *reinterpret_cast<volatile int*>(&q_unit[qslot]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&q_empty[qslot]);
        if (++qslot == kUnitQueue) {
            qslot = 0;
            qphase ^= 1;
        }
        return nxt;
    };

    if (warp >= CW) {
        // ================= TMA warpgroup (warps 8-11 / NAR 4-7; one lane issues) =
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
        if (warp != CW || lane != 0) return;
        uint32_t s = 0, phase = 0;
        for (int unit = blockIdx.x; unit < n_units; unit = producer_next(unit)) {
        const Unit U = decode_unit<GROUPS>(P, unit);
        const int m0 = U.tm * kBM, n0 = U.tn * BN;
        const int kt_lo = U.kt_lo, kt_hi = U.kt_hi;
        for (int p = U.p_lo; p < U.p_hi; ++p) {
            const ProductDesc& pd = P.prod[p];
            if (!NAR && pd.half) {
                // 8-k half tiles, two terms per slot (A terms first, then B)
                const int nt = pd.na + pd.nb;
                for (int kh = 2 * kt_lo; kh < 2 * kt_hi; ++kh) {
                    const int k0 = kh * (kBK / 2);
                    for (int u = 0; u < nt; u += 2) {
                        mbar_wait(&raw_empty[s], phase ^ 1);
                        mbar_expect_tx(&raw_full[s], (u + 1 < nt ? 2 : 1) * kHalfBytes);
                        for (int e = 0; e < 2 && u + e < nt; ++e) {
                            uint8_t* dst = raw + s * kSlotBytes + e * kHalfBytes;
                            const int t = u + e;
                            if (t < pd.na) {
                                const CUtensorMap* map = &P.tmAh[pd.aq[t]];
#pragma unroll
                                for (int box = 0; box < kBM / 16; ++box)
                                    tma_load_2d(dst + box * 1024, map, m0 + 16 * box, k0,
                                                &raw_full[s]);
                            } else {
                                tma_load_2d(dst, &P.tmBh[pd.bq[t - pd.na]], k0, n0, &raw_full[s]);
                            }
                        }
                        if (++s == RING) {
                            s = 0;
                            phase ^= 1;
                        }
                    }
                }
                continue;
            }
            for (int kt = kt_lo; kt < kt_hi; ++kt) {
                const int k0 = kt * kBK;
                for (int u = 0; u < pd.na + pd.nb; ++u) {
                    mbar_wait(&raw_empty[s], phase ^ 1);
                    // (a narrow B tile is 16 x 64: half a slot)
                    mbar_expect_tx(&raw_full[s], NAR && u >= pd.na ? kSlotBytes / 2 : kSlotBytes);
                    uint8_t* dst = raw + s * kSlotBytes;
                    if (u < pd.na) {
                        const CUtensorMap* map = &P.tmA[pd.aq[u]];
#pragma unroll
                        for (int box = 0; box < kBM / 16; ++box)
                            tma_load_2d(dst + box * 2048, map, m0 + 16 * box, k0, &raw_full[s]);
                    } else {
                        tma_load_2d(dst, &P.tmB[pd.bq[u - pd.na]], k0, n0, &raw_full[s]);
                    }
                    if (++s == RING) {
                        s = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        }  // unit
        return;
    }

    // ================= DMMA warpgroups (warps 0-7) ==========================
    // Each warp forms the Strassen operand sums of exactly the fragments it
    // multiplies, in registers, straight from the TMA term tiles: the sums'
    // DADDs sit in the DMMA warp's own instruction stream (DADDs issued by
    // other warps are starved while DMMA saturates the FP64 pipe, measured in
    // microbench/fp64_contend.cu), and no stage buffer, barrier or
    // cross-warp handoff is needed.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(NAR ? kNarrowConsumerRegs : kConsumerRegs));
    const int wm = warp & 1, wn = warp >> 1;
    const int g = lane >> 2, j = lane & 3;
    double acc[8][4][2];
    // ring position of the next term tile: slot index and its fill parity
    uint32_t slot = 0, phase = 0;
    // SEP: bulk reductions of the previous unit still in flight, and the ticket
    // (and product) to release once they complete
    bool pend = false;
    int pend_p = -1, pend_tm = 0, pend_tn = 0;  // pend_p >= 0: tickets to release
    // Completion of a unit's reduce-adds: a ticket successor needs them performed
    // (wait_group 0); otherwise only the stage must be free again (wait_group.read:
    // the writes complete before the grid does, as TMA stores do)
    auto collect = [&]() {  // every warp's reductions performed, then hand the tiles on
        if (pend_p >= 0) {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
        } else {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        consumer_bar<CW>();  // (also: the stage is free again)
        if (threadIdx.x == 0 && pend_p >= 0) {
            __threadfence();
            release_ticket(P, pend_p, pend_tm, pend_tn);
        }
        pend = false;
    };

    trace_event(P, 0);
    int trace_i = 0;
    for (int unit = blockIdx.x; unit < n_units; unit = consumer_next(unit)) {
    trace_event(P, 1 + 2 * trace_i);
    const Unit U = decode_unit<GROUPS>(P, unit);
    const int tm = U.tm, tn = U.tn, p_lo = U.p_lo, p_hi = U.p_hi;
    const int kt_lo = U.kt_lo, kt_hi = U.kt_hi;
    for (int p = p_lo; p < p_hi; ++p) {
        const ProductDesc& pd = P.prod[p];
        const int na = pd.na, nb = pd.nb;
        const bool neg_a0 = pd.as[0] < 0, neg_b0 = pd.bs[0] < 0;  // warp-uniform
        double ca[MAXT], cb[MAXT];
#pragma unroll
        for (int u = 0; u < MAXT; ++u) {
            ca[u] = u < na ? static_cast<double>(pd.as[u]) : 0.0;
            cb[u] = u < nb ? static_cast<double>(pd.bs[u]) : 0.0;
        }
#pragma unroll
        for (int mf = 0; mf < 8; ++mf)
#pragma unroll
            for (int nf = 0; nf < 4; ++nf) acc[mf][nf][0] = acc[mf][nf][1] = 0.0;

        // compile-time term counts for the combinations the tables produce
        // (1, 2 or 4 terms per side); anything else (clipped quadrants drop
        // terms) takes the generic loop
        const int combo = na * 8 + nb;
        bool done = true;
        if (combo == 9) {
            product_kloop<1, 1, RING>(raw, raw_full, raw_empty, slot, phase, kt_lo, kt_hi, pd, wm, wn,
                                g, j, lane, acc);
        } else if (MAXT >= 2 && combo == 10) {
            product_kloop<1, (MAXT >= 2 ? 2 : 1), RING>(raw, raw_full, raw_empty, slot, phase, kt_lo,
                                                  kt_hi, pd, wm, wn, g, j, lane, acc);
        } else if (!PERSIST && MAXT >= 2 && combo == 17 && P.a_heavy_layout) {
            product_kloop1<(MAXT >= 2 ? 2 : 1), 1, RING>(raw, raw_full, raw_empty, slot, phase,
                                                   kt_lo, kt_hi, pd, warp & 3, warp >> 2, g, j,
                                                   lane, acc);
            relayout_to_2x4(raw, acc, warp, g, j);
        } else if (MAXT >= 2 && combo == 17) {
            product_kloop<(MAXT >= 2 ? 2 : 1), 1, RING>(raw, raw_full, raw_empty, slot, phase, kt_lo,
                                                  kt_hi, pd, wm, wn, g, j, lane, acc);
        } else if (MAXT >= 2 && combo == 18) {
            product_kloop<(MAXT >= 2 ? 2 : 1), (MAXT >= 2 ? 2 : 1), RING>(
                raw, raw_full, raw_empty, slot, phase, kt_lo, kt_hi, pd, wm, wn, g, j, lane, acc);
        } else if (MAXT >= 4 && combo == 12) {
            product_kloop<1, (MAXT >= 4 ? 4 : 1), RING>(raw, raw_full, raw_empty, slot, phase, kt_lo,
                                                  kt_hi, pd, wm, wn, g, j, lane, acc);
        } else if (!PERSIST && MAXT >= 4 && combo == 33 && P.a_heavy_layout) {
            product_kloop1<(MAXT >= 4 ? 4 : 1), 1, RING>(raw, raw_full, raw_empty, slot, phase,
                                                   kt_lo, kt_hi, pd, warp & 3, warp >> 2, g, j,
                                                   lane, acc);
            relayout_to_2x4(raw, acc, warp, g, j);
        } else if (MAXT >= 4 && combo == 33) {
            product_kloop<(MAXT >= 4 ? 4 : 1), 1, RING>(raw, raw_full, raw_empty, slot, phase, kt_lo,
                                                  kt_hi, pd, wm, wn, g, j, lane, acc);
        } else if (MAXT >= 4 && combo == 20) {
            product_kloop<(MAXT >= 4 ? 2 : 1), (MAXT >= 4 ? 4 : 1), RING>(
                raw, raw_full, raw_empty, slot, phase, kt_lo, kt_hi, pd, wm, wn, g, j, lane, acc);
        } else if (!PERSIST && MAXT >= 4 && combo == 34 && P.a_heavy_layout) {
            product_kloop1<(MAXT >= 4 ? 4 : 1), (MAXT >= 4 ? 2 : 1), RING>(
                raw, raw_full, raw_empty, slot, phase, kt_lo, kt_hi, pd, warp & 3, warp >> 2, g, j,
                lane, acc);
            relayout_to_2x4(raw, acc, warp, g, j);
        } else if (MAXT >= 4 && combo == 34) {
            product_kloop<(MAXT >= 4 ? 4 : 1), (MAXT >= 4 ? 2 : 1), RING>(
                raw, raw_full, raw_empty, slot, phase, kt_lo, kt_hi, pd, wm, wn, g, j, lane, acc);
        } else if (MAXT >= 4 && combo == 36 && pd.half) {
            product_kloop_half<(MAXT >= 4 ? 4 : 1), (MAXT >= 4 ? 4 : 1), RING>(
                raw, raw_full, raw_empty, slot, phase, kt_lo, kt_hi, pd, wm, wn, g, j, lane, acc);
        } else if (MAXT >= 4 && combo == 36) {
            product_kloop<(MAXT >= 4 ? 4 : 1), (MAXT >= 4 ? 4 : 1), RING>(
                raw, raw_full, raw_empty, slot, phase, kt_lo, kt_hi, pd, wm, wn, g, j, lane, acc);
        } else {
            done = false;
        }
        if (!done)
        for (int kt = kt_lo; kt < kt_hi; ++kt) {
            // term tiles of this k-step: A terms, then B terms, in ring order
            // (a k-step uses at most 2*MAXT <= 8 < RING slots: one wrap at most)
            const uint8_t* sA[MAXT];
            const uint8_t* sB[MAXT];
            const uint32_t slot0 = slot;
#pragma unroll
            for (int u = 0; u < MAXT; ++u) {
                uint32_t sa = slot0 + u, sb = slot0 + na + u;
                const uint32_t pa = (sa >= RING) ? phase ^ 1 : phase;
                const uint32_t pb = (sb >= RING) ? phase ^ 1 : phase;
                sa = (sa >= RING) ? sa - RING : sa;
                sb = (sb >= RING) ? sb - RING : sb;
                sA[u] = raw + sa * kSlotBytes;
                sB[u] = raw + sb * kSlotBytes;
                if (u < na) mbar_wait(&raw_full[sa], pa);
                if (u < nb) mbar_wait(&raw_full[sb], pb);
            }
            slot += na + nb;
            if (slot >= RING) {
                slot -= RING;
                phase ^= 1;
            }
#pragma unroll
            for (int sp = 0; sp < 2; ++sp) {
                Frags f;
                frag_a_term<true>(sA[0], sp, wm, g, j, 1.0, f);
                frag_b_term<true>(sB[0], sp, wn, g, j, 1.0, f);
                if (neg_a0) {
#pragma unroll
                    for (int ss = 0; ss < 2; ++ss)
#pragma unroll
                        for (int mf = 0; mf < 8; ++mf) f.a[ss][mf] = -f.a[ss][mf];
                }
                if (neg_b0) {
#pragma unroll
                    for (int ss = 0; ss < 2; ++ss)
#pragma unroll
                        for (int nf = 0; nf < 4; ++nf) f.b[ss][nf] = -f.b[ss][nf];
                }
#pragma unroll
                for (int u = 1; u < MAXT; ++u) {
                    if (u < na) frag_a_term<false>(sA[u], sp, wm, g, j, ca[u], f);
                    if (u < nb) frag_b_term<false>(sB[u], sp, wn, g, j, cb[u], f);
                }
                dmma_substep(f, 0, acc);
                dmma_substep(f, 1, acc);
            }
            consumer_fence();
            __syncwarp();
            if (lane == 0) {
                uint32_t s2 = slot0;
                for (int u = 0; u < na + nb; ++u) {
                    mbar_arrive(&raw_empty[s2]);
                    if (++s2 == RING) s2 = 0;
                }
            }
        }

        // product groups: the first products of a group wait in tensor memory for the last
        if constexpr (GROUPS) {
            if (p + 1 < p_hi) {
                tmem_park(tmem_base, warp, p - p_lo, acc);
                continue;
            }
        }
        const bool paired = GROUPS && p_hi - p_lo >= 2;
        trace_event(P, 2 + 2 * trace_i);
        if (SEP && pend) collect();  // previous unit's reductions: complete, release its ticket
        // ---- epilogue of product p.  Accumulator (mf, nf, e) of lane (g, j)
        // is row 16(mf/2) + 2g + mf%2 and column 8nf + nperm(2j + e) of this
        // warp's 64 x 32 tile.
        const int mrow0 = tm * kBM + wm * 64 + 2 * g;
        const int ncol0 = tn * BN + wn * 32;
        // (half-tile products map B columns without the permutation)
        const int c0 = pd.half ? 2 * j : nperm(2 * j), c1 = pd.half ? 2 * j + 1 : nperm(2 * j + 1);
        // ---- fused epilogue through bulk reductions.  The DMMA warps stage
        // (alpha gamma) M in shared memory (the ring is idle once this CTA's
        // only product is done) and warp 0 hands each C column to the TMA
        // engine as an f64 add performed at L2 (cp.reduce.async.bulk): C never
        // passes through the SM and the warps do not wait on HBM.  Per element
        // the result is C + round(alpha gamma M) -- with |alpha| = 1 exactly the
        // fma(alpha gamma, M, C) of the register path.  Used for whole,
        // column-major tiles of single-product CTAs with short k loops (the
        // CTA stays resident until its reductions complete, which costs more
        // than the register path saves once the mainloop is long); anything
        // else takes the register read-modify-write below.
        // C tiles are reduced through the quadrants' tensor maps (tmC), which clip
        // partial tiles at the quadrant edge.
        bool bulk = !NAR && P.mode == kEpiRMW && P.c_tma && (p_hi - p_lo == 1 || GROUPS) &&
                    kt_hi - kt_lo <= P.bulk_max_kt && (SEP || !persistent) &&
                    U.npieces == 1;
        // the reduce-add clips rows at 16-byte granularity (microbench/tma_reduce_f64.cu):
        // a tile ending inside a quadrant with an odd row count takes the register path
        for (int u = 0; u < pd.nc && bulk; ++u) {
            const int R = P.crows[pd.cq[u]];
            bulk = (R & 1) == 0 || tm * kBM + kBM <= R;
        }
        // destinations of the unit and their coefficients on the parked products (da:
        // slot 0, dc: slot 1) and on the accumulator (db); a product alone has da = dc = 0
        // (GROUPS only: the other instantiations keep the single-product epilogue below)
        constexpr int kMaxDest = GROUPS ? (kParkSlots + 1) * kMaxTerms : 1;
        int nd = 0;
        int dq[kMaxDest];
        int8_t da[kMaxDest], db[kMaxDest], dc[kMaxDest];
        if constexpr (GROUPS) {
            for (int pp = paired ? p_lo : p; pp <= p; ++pp) {
                const ProductDesc& px = P.prod[pp];
                const int k = pp == p ? 2 : pp - p_lo;  // slot 0, slot 1, accumulator
                for (int u = 0; u < px.nc; ++u) {
                    int i = 0;
                    while (i < nd && dq[i] != px.cq[u]) ++i;
                    if (i == nd) {
                        dq[nd] = px.cq[u];
                        da[nd] = db[nd] = dc[nd] = 0;
                        ++nd;
                    }
                    (k == 0 ? da : k == 1 ? dc : db)[i] = px.cs[u];
                }
            }
            for (int i = 0; i < nd && bulk; ++i) {  // (the first products' destinations too)
                const int R = P.crows[dq[i]];
                bulk = (R & 1) == 0 || tm * kBM + kBM <= R;
            }
        }
        if (bulk) {
            // stage: 8 boxes of 16 rows x 128 columns (16 KB each, 128-byte swizzle:
            // column c at c*128, 16-byte chunk (row%16)/2 ^ c%8) -- conflict-free for
            // the fragment layout (chunk g ^ nperm(2j+e)%8 covers all 8 per quarter-warp)
            uint8_t* stage = SEP ? raw + RING * kSlotBytes + 1024 : raw;
            const bool ticketed = P.tickets != nullptr;
            bool issued = false;
            if (!SEP) consumer_bar<CW>();  // every warp is done reading the ring before it is reused
            // DMMA warp w hands box w (rows 16w..16w+15) of every destination to the TMA
            // engine: one tensor reduce-add each (per-column 1-D bulk reductions issued
            // 128 x nc uniform-datapath instructions per tile)
            static_assert(kConsumerWarps * 16 == kBM, "one 16-row box per warp");
            if constexpr (GROUPS) {
                // one pass per distinct (da, dc, db): stage alpha (da M0 + dc M1 + db M), then
                // one reduce-add per destination with those coefficients
                int done = 0;  // destinations already issued (bit mask)
                for (int first = 0; first < nd; ++first) {
                    if (done & (1 << first)) continue;
                    const int ca = da[first], cb = db[first], cc = dc[first];
                    if (issued) {  // previous pass's reductions must have read the stage
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        consumer_bar<CW>();
                    }
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        double v[16];
                        group_values(tmem_base, warp, h, ca, cc, cb, acc, v);
#pragma unroll
                        for (int nf = 0; nf < 4; ++nf)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int col = wn * 32 + 8 * nf + (e ? c1 : c0);
                                *reinterpret_cast<double2*>(stage + (wm * 4 + h) * 16384 + col * 128 +
                                                            ((g ^ (col & 7)) << 4)) =
                                    make_double2(P.alpha * v[2 * nf + e], P.alpha * v[8 + 2 * nf + e]);
                            }
                    }
                    consumer_fence();  // generic smem writes before the async-proxy reads
                    if (!issued && ticketed) {
                        trace_event(P, 20);  // (single-unit launches: first stage written)
                        if (threadIdx.x == 0) wait_ticket(P, U.tk, tm, tn);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        trace_event(P, 21);  // ticket held
                    }
                    consumer_bar<CW>();
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    for (int i = first; i < nd; ++i) {
                        if (da[i] != ca || db[i] != cb || dc[i] != cc) continue;
                        done |= 1 << i;
                        if (lane == 0)
                            tma_reduce_add_2d(&P.tmC[dq[i]], tm * kBM + 16 * warp, tn * kBN,
                                              stage + warp * 16384);
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    issued = true;
                }
            } else {
                for (int pass = 0; pass < 2; ++pass) {  // destinations with coefficient +1, then -1
                    int any = 0;
                    for (int u = 0; u < pd.nc; ++u) any |= (pd.cs[u] > 0) == (pass == 0);
                    if (!any) continue;
                    if (issued) {  // previous pass's reductions must have read the stage
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        consumer_bar<CW>();
                    }
                    const double sc = P.alpha * (pass == 0 ? 1.0 : -1.0);
#pragma unroll
                    for (int nf = 0; nf < 4; ++nf)
#pragma unroll
                        for (int h = 0; h < 4; ++h)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int col = wn * 32 + 8 * nf + (e ? c1 : c0);
                                *reinterpret_cast<double2*>(stage + (wm * 4 + h) * 16384 + col * 128 +
                                                            ((g ^ (col & 7)) << 4)) =
                                    make_double2(sc * acc[2 * h][nf][e], sc * acc[2 * h + 1][nf][e]);
                            }
                    consumer_fence();  // generic smem writes before the async-proxy reads
                    if (!issued && ticketed) {
                        if (threadIdx.x == 0) wait_ticket(P, U.tk, tm, tn);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    consumer_bar<CW>();
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    if (lane == 0) {
                        for (int u = 0; u < pd.nc; ++u) {
                            if ((pd.cs[u] > 0) != (pass == 0)) continue;
                            tma_reduce_add_2d(&P.tmC[pd.cq[u]], tm * kBM + 16 * warp, tn * kBN,
                                              stage + warp * 16384);
                        }
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    issued = true;
                }
            }
            // the last product (pair) of the launch has no ticket successor
            const bool succ = ticketed && U.tk + 1 < (GROUPS ? P.npairs : P.nprod);
            if (SEP && P.sep_defer) {  // completion collected at the next epilogue (or after the loop)
                pend = true;
                pend_p = succ ? U.tk : -1;
                pend_tm = tm;
                pend_tn = tn;
                continue;
            }
            trace_event(P, 22);  // every reduce-add issued
            if (succ) {  // all reductions performed (every warp's), then hand the tile on
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");
                consumer_bar<CW>();
                trace_event(P, 23);  // reductions complete
                if (threadIdx.x == 0) {
                    __threadfence();
                    release_ticket(P, U.tk, tm, tn);
                }
            } else {  // the stage must outlive the reads (smem is freed at exit)
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                consumer_bar<CW>();
            }
            continue;  // next product (none: single-product CTA)
        }
        if (GROUPS && paired) {
            // ---- a group's update through registers (C layouts the reduce-adds cannot
            // take): C += alpha (da Mparked + db M) per destination, in pair order --
            // per element the same arithmetic as the staged values of the bulk path
            if (P.tickets) {
                if (threadIdx.x == 0) wait_ticket(P, U.tk, tm, tn);
                consumer_bar<CW>();
            }
            for (int i = 0; i < nd; ++i) {
                double* __restrict__ C = P.cptr[dq[i]];
                const int R = P.crows[dq[i]], Cc = P.ccols[dq[i]];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    double v[16];
                    group_values(tmem_base, warp, h, da[i], dc[i], db[i], acc, v);
#pragma unroll
                    for (int nf = 0; nf < 4; ++nf)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const double v0 = v[2 * nf + e], v1 = v[8 + 2 * nf + e];
                            const int row = mrow0 + 16 * h;
                            const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                            if (col >= Cc) continue;
                            if (row < R) {
                                double* x = C + row * P.rs_c + static_cast<long long>(col) * P.cs_c;
                                *x = fma(P.alpha, v0, __ldcg(x));
                            }
                            if (row + 1 < R) {
                                double* x = C + (row + 1) * P.rs_c + static_cast<long long>(col) * P.cs_c;
                                *x = fma(P.alpha, v1, __ldcg(x));
                            }
                        }
                }
            }
            if (P.tickets) {  // every thread's C stores visible, then hand the tile on
                __threadfence();
                consumer_bar<CW>();
                if (threadIdx.x == 0) release_ticket(P, U.tk, tm, tn);
            }
            continue;
        }
        if (P.arrive && U.npieces > 1) {
            // ---- k-split / stream-K fixup: partials out, one piece sums them ----
            // (partials in slots p * ksplit + piece; ksplit = slots per product); the RMW
            // epilogue or (sk_store) the store of M_p follows.  M_p = P_0 + P_1 + ... in
            // piece (k) order, the stream pass's order.
            // Stream-K: piece 0 finishes the unit.  Its CTA reaches it last (a unit's head
            // lies at the end of one CTA's range, its other pieces at the start of the
            // next CTAs'), keeps its own partial in registers and waits for the others --
            // safe because every stream-K CTA is resident and a non-zero piece never waits.
            // k-chunk grids (CTAs may run in waves): the last piece to arrive sums them.
            const int s_idx = U.piece;
            const long long ldm = P.ldm;
            int* cnt = P.arrive + (tm * P.ticket_ld + tn) * P.nprod + p;
            // Cooperative fixup (MMParams::coop_fixup) when two or more pieces end
            // their CTAs' ranges: every piece stores its partial and coop_finish (not
            // inlined: the accumulators are dead by then, and code inlined here costs
            // the k-loops registers) shares the sums and the epilogue among them.
            int part_i = 0, nparts = 1;
            if (!GROUPS && P.coop_fixup) coop_participants(P, unit, s_idx, U.npieces, part_i, nparts);
            const bool coop = nparts >= 2;
            const bool owner0 = !coop && P.streamk && s_idx == 0;
            if (!owner0) {
                double* Mo = P.mbase + P.part_off +
                             static_cast<long long>(p * P.ksplit + s_idx) * P.mstride;
#pragma unroll
                for (int nf = 0; nf < 4; ++nf)
#pragma unroll
                    for (int h = 0; h < 4; ++h)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int row = mrow0 + 16 * h;
                            const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                            if (col >= P.qn || row >= P.qm) continue;
                            double* dst = Mo + row + static_cast<long long>(col) * ldm;
                            __stcg(reinterpret_cast<double2*>(dst),
                                   make_double2(acc[2 * h][nf][e], acc[2 * h + 1][nf][e]));
                        }
                __threadfence();
                consumer_bar<CW>();
            }
            if (coop) {
                // arrive; a participant (always its CTA's last unit) finishes its share
                // after the unit loop, where no loop state is live (coop_finish)
                if (threadIdx.x == 0) {
                    atomicAdd(cnt, 1);
                    if (part_i >= 0) {
                        coop_job[0] = 1;
                        coop_job[1] = p;
                        coop_job[2] = tm;
                        coop_job[3] = tn;
                        coop_job[4] = part_i;
                        coop_job[5] = nparts;
                        coop_job[6] = U.npieces;
                        coop_job[7] = pd.half;
                    }
                }
                continue;
            }
            __shared__ int last_flag;
            if (owner0) {  // wait for pieces 1 .. npieces - 1
                if (threadIdx.x == 0) {
                    while (ld_relaxed_gpu(cnt) != U.npieces - 1) __nanosleep(64);
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
                consumer_bar<CW>();
            } else {
                if (threadIdx.x == 0) {
                    const int before = atomicAdd(cnt, 1);
                    last_flag = !P.streamk && before == U.npieces - 1;
                }
                consumer_bar<CW>();
                if (!last_flag) continue;  // another piece finishes this product
                __threadfence();
            }
            // the other pieces' partials, read back from L2 and added in piece order
            // (piece 0's own partial is its accumulator)
            const double* Mp = P.mbase + P.part_off + static_cast<long long>(p * P.ksplit) * P.mstride;
            for (int sp = owner0 ? 1 : 0; sp < U.npieces; ++sp) {
#pragma unroll
                for (int nf = 0; nf < 4; ++nf)
#pragma unroll
                    for (int h = 0; h < 4; ++h)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int row = mrow0 + 16 * h;
                            const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                            double2 x = make_double2(0.0, 0.0);
                            if (col < P.qn && row < P.qm)
                                x = __ldcg(reinterpret_cast<const double2*>(
                                    Mp + static_cast<long long>(sp) * P.mstride + row +
                                    static_cast<long long>(col) * ldm));
                            if (sp == 0) {
                                acc[2 * h][nf][e] = x.x;
                                acc[2 * h + 1][nf][e] = x.y;
                            } else {
                                acc[2 * h][nf][e] += x.x;
                                acc[2 * h + 1][nf][e] += x.y;
                            }
                        }
            }
        }
        const bool ticketed = P.mode == kEpiRMW && P.tickets;  // ordered epilogue
        if (ticketed) {
            if (threadIdx.x == 0) wait_ticket(P, U.tk, tm, tn);
            consumer_bar<CW>();
        }
        if (P.mode == kEpiRMW) {
            // 16-byte path: C column-major with rows (2g, 2g+1) of the fragment
            // pair (2h, 2h+1) adjacent and 16-byte aligned (checked on the host)
            for (int u = 0; u < pd.nc; ++u) {
                const int cq = pd.cq[u];
                double* __restrict__ C = P.cptr[cq];
                const int R = P.crows[cq], Cc = P.ccols[cq];
                const double sc = P.alpha * static_cast<double>(pd.cs[u]);
                if (P.c_vec) {
#pragma unroll
                    for (int nh = 0; nh < 2; ++nh) {  // two rounds of 16 loads in flight
                        double2 cv[2][4][2];
#pragma unroll
                        for (int n2 = 0; n2 < 2; ++n2)
#pragma unroll
                            for (int h = 0; h < 4; ++h)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int nf = 2 * nh + n2;
                                    const int row = mrow0 + 16 * h;
                                    const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                                    double2 v = make_double2(0.0, 0.0);
                                    if (col < Cc) {
                                        const double* src = C + row + static_cast<long long>(col) * P.cs_c;
                                        if (row + 1 < R) v = __ldcg(reinterpret_cast<const double2*>(src));
                                        else if (row < R) v.x = __ldcg(src);
                                    }
                                    cv[n2][h][e] = v;
                                }
#pragma unroll
                        for (int n2 = 0; n2 < 2; ++n2)
#pragma unroll
                            for (int h = 0; h < 4; ++h)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int nf = 2 * nh + n2;
                                    const int row = mrow0 + 16 * h;
                                    const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                                    if (col >= Cc) continue;
                                    double* dst = C + row + static_cast<long long>(col) * P.cs_c;
                                    double2 v = cv[n2][h][e];
                                    v.x = fma(sc, acc[2 * h][nf][e], v.x);
                                    v.y = fma(sc, acc[2 * h + 1][nf][e], v.y);
                                    if (row + 1 < R) *reinterpret_cast<double2*>(dst) = v;
                                    else if (row < R) *dst = v.x;
                                }
                    }
                    continue;
                }
#pragma unroll
                for (int nf = 0; nf < 4; ++nf) {
                    double cv[8][2];
#pragma unroll
                    for (int mf = 0; mf < 8; ++mf)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int row = mrow0 + 16 * (mf >> 1) + (mf & 1);
                            const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                            cv[mf][e] = (row < R && col < Cc)
                                            ? __ldcg(C + row * P.rs_c + col * P.cs_c) : 0.0;
                        }
#pragma unroll
                    for (int mf = 0; mf < 8; ++mf)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int row = mrow0 + 16 * (mf >> 1) + (mf & 1);
                            const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                            if (row < R && col < Cc)
                                C[row * P.rs_c + col * P.cs_c] = fma(sc, acc[mf][nf][e], cv[mf][e]);
                        }
                }
            }
            if (ticketed) {  // every thread's C stores visible, then hand the tiles on
                __threadfence();
                consumer_bar<CW>();
                if (threadIdx.x == 0) release_ticket(P, U.tk, tm, tn);
            }
        } else {
            const int mi = P.sk_store ? p : P.split ? p * P.ksplit + U.piece : p;
            // product temporaries: rows 2g, 2g+1 of fragment pair (2h, 2h+1)
            // are adjacent (ldm even) -> one 16-byte streaming store
            // (st.global.cs: evict-first, keeps operand panels in L2)
            double* __restrict__ M = P.mbase + mi * P.mstride;
#pragma unroll
            for (int nf = 0; nf < 4; ++nf)
#pragma unroll
                for (int h = 0; h < 4; ++h)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int row = mrow0 + 16 * h;
                        const int col = ncol0 + 8 * nf + (e ? c1 : c0);
                        if (col >= P.qn) continue;
                        double* dst = M + row + static_cast<long long>(col) * P.ldm;
                        if (row + 1 < P.qm) {
                            asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(dst),
                                         "d"(acc[2 * h][nf][e]), "d"(acc[2 * h + 1][nf][e])
                                         : "memory");
                        } else if (row < P.qm) {
                            dst[0] = acc[2 * h][nf][e];
                        }
                    }
        }
    }
    ++trace_i;
    }  // unit
    if (SEP && pend) collect();
    if constexpr (!GROUPS) {  // (product groups never split k)
    consumer_bar<CW>();  // (coop_job written by thread 0)
    if (coop_job[0]) {
        const int p = coop_job[1], tm = coop_job[2], tn = coop_job[3];
        const int mrow0 = tm * kBM + wm * 64 + 2 * g;
        const int ncol0 = tn * BN + wn * 32;
        const int c0 = coop_job[7] ? 2 * j : nperm(2 * j), c1 = coop_job[7] ? 2 * j + 1 : nperm(2 * j + 1);
        coop_finish<CW>(P, P.prod[p], p, tm, tn, mrow0, ncol0, c0, c1, warp, coop_job[4], coop_job[5],
                        coop_job[6]);
    }
    }
    trace_event(P, 31);
    if constexpr (GROUPS) {  // every warp is done with tensor memory; warp 0 frees it
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        consumer_bar<CW>();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "n"(kTmemCols)
                         : "memory");
    }
}

// ---------------------------------------------------------------- repack ----
__global__ void repack_kernel(const double* __restrict__ src, long long rs, long long cs,
                              long rows, long cols, double* __restrict__ dst, long long ld,
                              long q, long q_al, int x_along_rows) {
    __shared__ double tile[32][33];
    const long i0 = static_cast<long>(blockIdx.x) * 32;
    const long j0 = static_cast<long>(blockIdx.y) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    if (x_along_rows) {
        for (int yy = ty; yy < 32; yy += 8) {
            const long i = i0 + tx, jj = j0 + yy;
            if (i < rows && jj < cols) tile[yy][tx] = src[i * rs + jj * cs];
        }
    } else {
        for (int yy = ty; yy < 32; yy += 8) {
            const long i = i0 + yy, jj = j0 + tx;
            if (i < rows && jj < cols) tile[tx][yy] = src[i * rs + jj * cs];
        }
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
        const long i = i0 + tx, jj = j0 + yy;
        if (i < rows && jj < cols) {
            const long di = (i / q) * q_al + i % q;
            dst[di + jj * ld] = tile[yy][tx];
        }
    }
}

// ------------------------------------------- sum and stream passes (gather) ---
// A level-2 side has 16 quadrants feeding 45 operand sums (185 term reads if
// each sum read its own terms).  The gather forms read every source ONCE per
// position, keep the values in shared memory (indexable; each thread touches
// only its own slots, so no barrier) and emit every output: HBM traffic =
// sources + outputs.
// Sum pass: materialize_sum (variants.cpp:53-96) for all entries at once,
// d0*x0 then += ds*xs in listed order per element.
// Stream pass: C_r += (alpha gamma) M_p (variants.cpp:99-109), each quadrant's
// updates in table order.
struct SumGatherParams {
    const double* src[kMaxQuad];
    int srows[kMaxQuad], scols[kMaxQuad];
    long long sld[kMaxQuad];
    int nsrc;
    double* dst[kMaxSumJobs];
    int8_t nterms[kMaxSumJobs];
    int8_t tsrc[kMaxSumJobs][kMaxTerms];
    int8_t tcoeff[kMaxSumJobs][kMaxTerms];
    int njobs;
    long long rows, cols, ld;
    long long r0, c0;
};
constexpr int kGatherThreads = 128;

__device__ __forceinline__ void gather_sources(const SumGatherParams& P, long long i, long long j,
                                               double2 (&x)[kMaxQuad]) {
#pragma unroll
    for (int q = 0; q < kMaxQuad; ++q) {
        x[q] = make_double2(0.0, 0.0);
        if (q < P.nsrc && j < P.scols[q]) {
            const double* px = P.src[q] + i + j * P.sld[q];
            if (i + 1 < P.srows[q])
                x[q] = *reinterpret_cast<const double2*>(px);
            else if (i < P.srows[q])
                x[q].x = *px;
        }
    }
}

__global__ void __launch_bounds__(kGatherThreads)
sum_gather_kernel(const __grid_constant__ SumGatherParams P) {
    __shared__ double2 xs[kMaxQuad][kGatherThreads];  // 32 KB
    const int tid = threadIdx.x;
    const long long i = P.r0 + 2 * (static_cast<long long>(blockIdx.x) * kGatherThreads + tid);
    long long j = P.c0 + blockIdx.y;
    if (i >= P.rows || j >= P.cols) return;
    const bool pair = i + 1 < P.rows;
    // the next column's sources are loaded while this column's sums are formed
    double2 nx[kMaxQuad];
    gather_sources(P, i, j, nx);
    for (; j < P.cols; j += gridDim.y) {
#pragma unroll
        for (int q = 0; q < kMaxQuad; ++q)
            if (q < P.nsrc) xs[q][tid] = nx[q];
        if (j + gridDim.y < P.cols) gather_sources(P, i, j + gridDim.y, nx);
        for (int z = 0; z < P.njobs; ++z) {
            const int n = P.nterms[z];
            const double c0 = P.tcoeff[z][0];
            const double2 x0 = xs[P.tsrc[z][0]][tid];
            double2 v = make_double2(c0 * x0.x, c0 * x0.y);
            for (int u = 1; u < n; ++u) {
                const double cu = P.tcoeff[z][u];
                const double2 x = xs[P.tsrc[z][u]][tid];
                v.x = fma(cu, x.x, v.x);
                v.y = fma(cu, x.y, v.y);
            }
            double* pd = P.dst[z] + i + j * P.ld;
            if (pair)
                *reinterpret_cast<double2*>(pd) = v;
            else
                *pd = v.x;
        }
    }
}

struct StreamGatherParams {
    double* cptr[kMaxQuad];
    int crows[kMaxQuad], ccols[kMaxQuad];
    long long rs_c, cs_c;
    int nquad;
    const double* mbase;
    long long mstride, ldm;
    int ksplit;
    int nprod;
    int8_t ndest[kMaxProducts];
    int8_t dq[kMaxProducts][kMaxQuad];
    int8_t dcoeff[kMaxProducts][kMaxQuad];
    double alpha;
    int qm, qn;
    int r0, r1, c0, c1;
    int c_vec;
};
constexpr int kStreamThreads = 256;
constexpr int kStreamBatch = 8;  // M loads in flight per thread

__global__ void __launch_bounds__(kStreamThreads)
stream_gather_kernel(const __grid_constant__ StreamGatherParams P) {
    __shared__ double cs[kMaxQuad][kStreamThreads];  // 32 KB
    const int tid = threadIdx.x;
    const long long i = P.r0 + static_cast<long long>(blockIdx.x) * kStreamThreads + tid;
    if (i >= P.r1) return;
    for (long long j = P.c0 + blockIdx.y; j < P.c1; j += gridDim.y) {
#pragma unroll
        for (int q = 0; q < kMaxQuad; ++q)
            if (q < P.nquad)
                cs[q][tid] = (i < P.crows[q] && j < P.ccols[q])
                                 ? P.cptr[q][i * P.rs_c + j * P.cs_c] : 0.0;
        const double* Mij = P.mbase + i + j * P.ldm;
        for (int p0 = 0; p0 < P.nprod; p0 += kStreamBatch) {
            double v[kStreamBatch];
#pragma unroll
            for (int t = 0; t < kStreamBatch; ++t) {
                if (p0 + t < P.nprod) {
                    const double* M = Mij + static_cast<long long>(p0 + t) * P.ksplit * P.mstride;
                    v[t] = M[0];
                    for (int sp = 1; sp < P.ksplit; ++sp) v[t] += M[sp * P.mstride];
                }
            }
#pragma unroll
            for (int t = 0; t < kStreamBatch; ++t) {
                if (p0 + t >= P.nprod) break;
                const int nd = P.ndest[p0 + t];
                for (int d = 0; d < nd; ++d) {
                    const int q = P.dq[p0 + t][d];
                    cs[q][tid] = fma(P.alpha * static_cast<double>(P.dcoeff[p0 + t][d]), v[t],
                                     cs[q][tid]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kMaxQuad; ++q)
            if (q < P.nquad && i < P.crows[q] && j < P.ccols[q])
                P.cptr[q][i * P.rs_c + j * P.cs_c] = cs[q][tid];
    }
}

// Row-pair form (C column-major with 16-byte aligned quadrants, even ldm):
// 16-byte loads and stores, otherwise identical per element.
constexpr int kStream2Threads = 128;

__global__ void __launch_bounds__(kStream2Threads)
stream_gather2_kernel(const __grid_constant__ StreamGatherParams P) {
    __shared__ double2 cs[kMaxQuad][kStream2Threads];  // 32 KB
    const int tid = threadIdx.x;
    const long long i = P.r0 + 2 * (static_cast<long long>(blockIdx.x) * kStream2Threads + tid);
    if (i >= P.r1) return;
    for (long long j = P.c0 + blockIdx.y; j < P.c1; j += gridDim.y) {
#pragma unroll
        for (int q = 0; q < kMaxQuad; ++q)
            if (q < P.nquad) {
                double2 c = make_double2(0.0, 0.0);
                if (j < P.ccols[q]) {
                    const double* pc = P.cptr[q] + i + j * P.cs_c;
                    if (i + 1 < P.crows[q])
                        c = *reinterpret_cast<const double2*>(pc);
                    else if (i < P.crows[q])
                        c.x = *pc;
                }
                cs[q][tid] = c;
            }
        const double* Mij = P.mbase + i + j * P.ldm;
        for (int p0 = 0; p0 < P.nprod; p0 += kStreamBatch) {
            double2 v[kStreamBatch];
#pragma unroll
            for (int t = 0; t < kStreamBatch; ++t) {
                if (p0 + t < P.nprod) {
                    const double* M = Mij + static_cast<long long>(p0 + t) * P.ksplit * P.mstride;
                    v[t] = *reinterpret_cast<const double2*>(M);
                    for (int sp = 1; sp < P.ksplit; ++sp) {
                        const double2 x = *reinterpret_cast<const double2*>(M + sp * P.mstride);
                        v[t].x += x.x;
                        v[t].y += x.y;
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < kStreamBatch; ++t) {
                if (p0 + t >= P.nprod) break;
                const int nd = P.ndest[p0 + t];
                for (int d = 0; d < nd; ++d) {
                    const int q = P.dq[p0 + t][d];
                    const double g = P.alpha * static_cast<double>(P.dcoeff[p0 + t][d]);
                    double2 c = cs[q][tid];
                    c.x = fma(g, v[t].x, c.x);
                    c.y = fma(g, v[t].y, c.y);
                    cs[q][tid] = c;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kMaxQuad; ++q)
            if (q < P.nquad && j < P.ccols[q]) {
                double* pc = P.cptr[q] + i + j * P.cs_c;
                if (i + 1 < P.crows[q])
                    *reinterpret_cast<double2*>(pc) = cs[q][tid];
                else if (i < P.crows[q])
                    *pc = cs[q][tid].x;
            }
    }
}

template <int L, int PR, int D>
__device__ __forceinline__ void stream_upd(double2 (&acc)[L == 1 ? 4 : 16], const double2& v,
                                           const StreamGatherParams& P) {
    if constexpr (D < stream_tab<L>().nd[PR]) {
        constexpr int q = stream_tab<L>().dq[PR][D];
        const double g = P.alpha * static_cast<double>(P.dcoeff[PR][D]);
        acc[q].x = fma(g, v.x, acc[q].x);
        acc[q].y = fma(g, v.y, acc[q].y);
        stream_upd<L, PR, D + 1>(acc, v, P);
    }
}

template <int L, int P0, int T = 0>
__device__ __forceinline__ void stream_apply(double2 (&acc)[L == 1 ? 4 : 16],
                                             const double2 (&v)[kStreamBatch],
                                             const StreamGatherParams& P) {
    if constexpr (T < kStreamBatch && P0 + T < stream_tab<L>().np) {
        stream_upd<L, P0 + T, 0>(acc, v[T], P);
        stream_apply<L, P0, T + 1>(acc, v, P);
    }
}

// products B*8 .. B*8+7: their M values loaded together, then applied in order.
// KS > 0: the k-split count is a compile-time constant, so all KS x 8 partial loads of
// a batch are issued before the first add (one memory round trip per batch instead of
// a chain of KS per product); the adds keep the split order, so the sums are bitwise
// the same as the runtime-KS form (KS = 0).
template <int L, int B, int KS>
__device__ __forceinline__ void stream_batch(double2 (&acc)[L == 1 ? 4 : 16], const double* Mij,
                                             const StreamGatherParams& P) {
    constexpr int NP = stream_tab<L>().np;
    if constexpr (B * kStreamBatch < NP && KS > 0) {
        double2 x[kStreamBatch][KS];
#pragma unroll
        for (int t = 0; t < kStreamBatch; ++t)
            if (B * kStreamBatch + t < NP) {
                const double* M = Mij + static_cast<long long>(B * kStreamBatch + t) * KS *
                                            P.mstride;
#pragma unroll
                for (int sp = 0; sp < KS; ++sp)
                    x[t][sp] = *reinterpret_cast<const double2*>(M + sp * P.mstride);
            }
        double2 v[kStreamBatch];
#pragma unroll
        for (int t = 0; t < kStreamBatch; ++t)
            if (B * kStreamBatch + t < NP) {
                v[t] = x[t][0];
#pragma unroll
                for (int sp = 1; sp < KS; ++sp) {
                    v[t].x += x[t][sp].x;
                    v[t].y += x[t][sp].y;
                }
            }
        stream_apply<L, B * kStreamBatch>(acc, v, P);
        stream_batch<L, B + 1, KS>(acc, Mij, P);
    } else if constexpr (B * kStreamBatch < NP) {
        double2 v[kStreamBatch];
#pragma unroll
        for (int t = 0; t < kStreamBatch; ++t) {
            if (B * kStreamBatch + t < NP) {
                const double* M = Mij + static_cast<long long>(B * kStreamBatch + t) * P.ksplit *
                                            P.mstride;
                v[t] = *reinterpret_cast<const double2*>(M);
                for (int sp = 1; sp < P.ksplit; ++sp) {
                    const double2 x = *reinterpret_cast<const double2*>(M + sp * P.mstride);
                    v[t].x += x.x;
                    v[t].y += x.y;
                }
            }
        }
        stream_apply<L, B * kStreamBatch>(acc, v, P);
        stream_batch<L, B + 1, KS>(acc, Mij, P);
    }
}

template <int L, int KS>
__global__ void __launch_bounds__(kStream2Threads)
stream_fixed_kernel(const __grid_constant__ StreamGatherParams P) {
    constexpr int NQ = L == 1 ? 4 : 16;
    const int tid = threadIdx.x;
    const long long i = P.r0 + 2 * (static_cast<long long>(blockIdx.x) * kStream2Threads + tid);
    if (i >= P.r1) return;
    for (long long j = P.c0 + blockIdx.y; j < P.c1; j += gridDim.y) {
        double2 acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            acc[q] = make_double2(0.0, 0.0);
            if (j < P.ccols[q]) {
                const double* pc = P.cptr[q] + i + j * P.cs_c;
                if (i + 1 < P.crows[q])
                    acc[q] = *reinterpret_cast<const double2*>(pc);
                else if (i < P.crows[q])
                    acc[q].x = *pc;
            }
        }
        stream_batch<L, 0, KS>(acc, P.mbase + i + j * P.ldm, P);
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if (j < P.ccols[q]) {
                double* pc = P.cptr[q] + i + j * P.cs_c;
                if (i + 1 < P.crows[q])
                    *reinterpret_cast<double2*>(pc) = acc[q];
                else if (i < P.crows[q])
                    *pc = acc[q].x;
            }
    }
}

// Does the gather form's (product -> destination quadrants) structure equal the
// level-L table?  (Coefficients stay runtime parameters.)
template <int L>
bool matches_stream_tab(const StreamGatherParams& g) {
    const StreamTab& t = stream_tab<L>();
    if (g.nquad != (L == 1 ? 4 : 16) || g.nprod != t.np) return false;
    for (int p = 0; p < t.np; ++p) {
        if (g.ndest[p] != t.nd[p]) return false;
        for (int d = 0; d < t.nd[p]; ++d)
            if (g.dq[p][d] != t.dq[p][d]) return false;
    }
    return true;
}

__global__ void scale_kernel(double* c, long rows, long cols, long long rs, long long cs,
                             double beta) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    for (long long j = blockIdx.y; j < cols; j += gridDim.y) {
        double* p = c + i * rs + j * cs;
        *p = (beta == 0.0) ? 0.0 : beta * *p;
    }
}

}  // namespace

template <int MAXT, bool PERSIST, int RING, bool GROUPS, bool NAR = false>
static cudaError_t launch_mm_g(const MMParams& p, cudaStream_t s);
template <int MAXT, bool PERSIST, int RING = kRawSlots>
static cudaError_t launch_mm_t(const MMParams& p, cudaStream_t s) {
    return p.pair_mode ? launch_mm_g<MAXT, PERSIST, RING, true>(p, s)
                       : launch_mm_g<MAXT, PERSIST, RING, false>(p, s);
}
template <int MAXT, bool PERSIST, int RING, bool GROUPS, bool NAR>
static cudaError_t launch_mm_g(const MMParams& p, cudaStream_t s) {
    constexpr int smem = NAR                ? kNarrowSmemBytes
                         : RING == kRawSlots ? kMMSmemBytes
                                             : mm_sep_smem_bytes(RING);
    // the > 48 KB dynamic shared-memory opt-in is per device context: once per device
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_set.load(std::memory_order_acquire) & bit)) {
        cudaError_t e = cudaFuncSetAttribute(mm_kernel<MAXT, PERSIST, RING, GROUPS, NAR>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(bit, std::memory_order_release);
    }
    const int units = p.tiles_m * p.tiles_n *
                      (p.pair_mode ? p.npairs : p.split ? p.nprod * p.ksplit : 1);
    // stream-K: exactly grid_cap CTAs (the unit decode assumes it)
    const int grid = PERSIST && p.streamk ? p.grid_cap
                     : PERSIST && p.grid_cap > 0 && p.grid_cap < units ? p.grid_cap : units;
    mm_kernel<MAXT, PERSIST, RING, GROUPS, NAR>
        <<<grid, NAR ? kNarrowThreads : kThreads, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_mm(const MMParams& p, cudaStream_t s) {
    int maxt = 1;
    for (int i = 0; i < p.nprod; ++i) {
        maxt = p.prod[i].na > maxt ? p.prod[i].na : maxt;
        maxt = p.prod[i].nb > maxt ? p.prod[i].nb : maxt;
    }
    // narrow tiles (small problems, two CTAs per SM): persistent, at most 2-term sums,
    // register epilogues (the host plans them so)
    if (p.narrow) {
        if (maxt > 2 || p.pair_mode || p.c_tma || p.sep_stage) return cudaErrorInvalidValue;
        return maxt == 1 ? launch_mm_g<1, true, kNarrowRing, false, true>(p, s)
                         : launch_mm_g<2, true, kNarrowRing, false, true>(p, s);
    }
    // Persistent launches for single-term programs (DGEMM, Naive, C): at 16384^3
    // mm_kernel 192.4 -> 188.7 ms (Naive L2), 251.4 -> 247.7 (DGEMM) on one box.
    // Fused-sum programs keep one CTA per unit: their units' costs differ by term
    // count and dynamic dispatch balances them better (ABC L1 233.8 vs 236.5 ms).
    if (maxt == 1 && p.grid_cap > 0 && p.sep_stage)  // persistent, deferred bulk epilogue
        return launch_mm_t<1, true, kSepRing>(p, s);
    if (maxt == 2 && p.grid_cap > 0 && p.sep_stage)  // the same with 2-term fused sums
        return launch_mm_t<2, true, kSepRing2>(p, s);
    if (maxt == 1)  // single-term programs: no sum code at all
        return p.grid_cap > 0 ? launch_mm_t<1, true>(p, s) : launch_mm_t<1, false>(p, s);
    if (p.streamk)  // stream-K of a fused-sum program (few tiles)
        return maxt <= 2 ? launch_mm_t<2, true>(p, s) : launch_mm_t<kMaxTerms, true>(p, s);
    return maxt <= 2 ? launch_mm_t<2, false>(p, s) : launch_mm_t<kMaxTerms, false>(p, s);
}

cudaError_t launch_repack(const double* src, long long rs, long long cs, long rows, long cols,
                          double* dst, long long ld, long q, long q_al, cudaStream_t s) {
    const long long ars = rs < 0 ? -rs : rs, acs = cs < 0 ? -cs : cs;
    const int x_along_rows = (ars <= acs) ? 1 : 0;
    dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
    repack_kernel<<<grid, dim3(32, 8), 0, s>>>(src, rs, cs, rows, cols, dst, ld, q, q_al,
                                               x_along_rows);
    return cudaGetLastError();
}

static unsigned col_grid(long long cols) {
    return static_cast<unsigned>(cols < 16384 ? cols : 16384);
}

// Gather form when the jobs draw on at most kMaxQuad distinct sources (every
// level-1/2 side); otherwise the per-job form.
static bool to_gather(const SumBatchParams& p, SumGatherParams& g) {
    std::memset(&g, 0, sizeof(g));
    for (int z = 0; z < p.njobs; ++z) {
        g.dst[z] = p.dst[z];
        g.nterms[z] = static_cast<int8_t>(p.nterms[z]);
        for (int u = 0; u < p.nterms[z]; ++u) {
            const SumTerm& t = p.t[z][u];
            int q = 0;
            while (q < g.nsrc && !(g.src[q] == t.x && g.srows[q] == t.rows &&
                                   g.scols[q] == t.cols && g.sld[q] == t.ld))
                ++q;
            if (q == g.nsrc) {
                if (g.nsrc == kMaxQuad) return false;
                g.src[q] = t.x;
                g.srows[q] = t.rows;
                g.scols[q] = t.cols;
                g.sld[q] = t.ld;
                ++g.nsrc;
            }
            g.tsrc[z][u] = static_cast<int8_t>(q);
            g.tcoeff[z][u] = static_cast<int8_t>(t.coeff);
        }
    }
    g.njobs = p.njobs;
    g.rows = p.rows;
    g.cols = p.cols;
    g.ld = p.ld;
    g.r0 = p.r0;
    g.c0 = p.c0;
    return true;
}

cudaError_t launch_sum_batch(const SumBatchParams& p, cudaStream_t s) {
    if (p.njobs == 0) return cudaSuccess;
    static thread_local SumGatherParams g;  // host staging; copied at launch
    if (to_gather(p, g)) {
        const long long pairs = (p.rows - p.r0 + 1) / 2;
        const long long w = p.cols - p.c0;
        dim3 grid(static_cast<unsigned>((pairs + kGatherThreads - 1) / kGatherThreads),
                  static_cast<unsigned>(w < 2048 ? w : 2048));
        sum_gather_kernel<<<grid, kGatherThreads, 0, s>>>(g);
        return cudaGetLastError();
    }
    return cudaErrorInvalidValue;  // > kMaxQuad distinct sources: not produced at L <= 2
}

// Product-major gather form: valid when every quadrant's sources are in
// ascending product order (table order), so visiting products in order applies
// each quadrant's updates in the same order as the per-quadrant form.
static bool to_gather(const StreamParams& p, StreamGatherParams& g) {
    std::memset(&g, 0, sizeof(g));
    for (int q = 0; q < p.nquad; ++q)
        for (int u = 0; u < p.nsrc[q]; ++u) {
            const int pr = p.src_prod[q][u];
            if (pr < 0 || pr >= kMaxProducts) return false;
            if (u > 0 && pr <= p.src_prod[q][u - 1]) return false;
            g.nprod = pr + 1 > g.nprod ? pr + 1 : g.nprod;
            g.dq[pr][g.ndest[pr]] = static_cast<int8_t>(q);
            g.dcoeff[pr][g.ndest[pr]] = p.src_coeff[q][u];
            ++g.ndest[pr];
        }
    for (int q = 0; q < kMaxQuad; ++q) {
        g.cptr[q] = p.cptr[q];
        g.crows[q] = p.crows[q];
        g.ccols[q] = p.ccols[q];
    }
    g.rs_c = p.rs_c;
    g.cs_c = p.cs_c;
    g.nquad = p.nquad;
    g.mbase = p.mbase;
    g.mstride = p.mstride;
    g.ldm = p.ldm;
    g.ksplit = p.ksplit;
    g.alpha = p.alpha;
    g.qm = p.qm;
    g.qn = p.qn;
    g.r0 = p.r0;
    g.r1 = p.r1;
    g.c0 = p.c0;
    g.c1 = p.c1;
    g.c_vec = p.c_vec;
    return true;
}

// register stream pass with the k-split count as a template constant where it is small
template <int L>
void launch_stream_fixed(dim3 grid, const StreamGatherParams& g, cudaStream_t s) {
    static const bool ks_on = [] {
        const char* v = std::getenv("STRASSEN_B200_STREAM_KS");  // 0 / 1 (experiments)
        return v ? std::atoi(v) != 0 : true;
    }();
    // level 1 only: at level 2 the 49 x KS loads in flight per thread measured slower
    // (2048^3 Naive L2 stream pass 56 -> 76 us, profiles/r01_stream_ks_probe.log); KS = 1
    // is the runtime form's schedule already
    if constexpr (L == 1) {
        switch (ks_on ? g.ksplit : 0) {
            case 2: stream_fixed_kernel<L, 2><<<grid, kStream2Threads, 0, s>>>(g); return;
            case 3: stream_fixed_kernel<L, 3><<<grid, kStream2Threads, 0, s>>>(g); return;
            case 4: stream_fixed_kernel<L, 4><<<grid, kStream2Threads, 0, s>>>(g); return;
            default: break;
        }
    }
    stream_fixed_kernel<L, 0><<<grid, kStream2Threads, 0, s>>>(g);
}

cudaError_t launch_stream_update(const StreamParams& p, cudaStream_t s) {
    static thread_local StreamGatherParams g;
    static const int ycap = [] {
        const char* v = std::getenv("STRASSEN_B200_STREAM_Y");  // grid.y cap (experiments)
        return v ? std::atoi(v) : 4096;
    }();
    if (to_gather(p, g)) {
        const int w = p.c1 - p.c0 < ycap ? p.c1 - p.c0 : ycap;
        if (p.c_vec && p.ldm % 2 == 0 && p.mstride % 2 == 0) {  // 16-byte rows pairs
            dim3 grid(static_cast<unsigned>(((p.r1 - p.r0 + 1) / 2 + kStream2Threads - 1) /
                                            kStream2Threads),
                      static_cast<unsigned>(w));
            static const bool fixed_on = [] {
                const char* v = std::getenv("STRASSEN_B200_STREAM_FIXED");  // 0 / 1 (experiments)
                return v ? std::atoi(v) != 0 : true;
            }();
            if (fixed_on && matches_stream_tab<2>(g))
                launch_stream_fixed<2>(grid, g, s);
            else if (fixed_on && matches_stream_tab<1>(g))
                launch_stream_fixed<1>(grid, g, s);
            else
                stream_gather2_kernel<<<grid, kStream2Threads, 0, s>>>(g);
            return cudaGetLastError();
        }
        dim3 grid(static_cast<unsigned>((p.r1 - p.r0 + kStreamThreads - 1) / kStreamThreads),
                  static_cast<unsigned>(w));
        stream_gather_kernel<<<grid, kStreamThreads, 0, s>>>(g);
        return cudaGetLastError();
    }
    return cudaErrorInvalidValue;  // per-quadrant lists not in table order: never built
}

cudaError_t launch_scale(double* c, long rows, long cols, long long rs, long long cs, double beta,
                         cudaStream_t s) {
    dim3 grid(static_cast<unsigned>((rows + 255) / 256), col_grid(cols));
    scale_kernel<<<grid, 256, 0, s>>>(c, rows, cols, rs, cs, beta);
    return cudaGetLastError();
}

}  // namespace sb200
