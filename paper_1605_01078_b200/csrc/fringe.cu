// Fringe updates of dynamic peeling (engine.cpp run_device): after the even core
// m_e x n_e x k_e has gone through Strassen, the three classical updates that finish
// C := alpha A B + C have one dimension of at most 16 (2^L - 1 <= 7 for odd sizes; up to
// 16 where the core is cut back to a whole number of quadrant tiles):
//   k fringe:  C[0:me, 0:ne] += alpha A[0:me, ke:k] B[ke:k, 0:ne]      (rank-kf update)
//   m fringe:  C[me:m, 0:n]  += alpha A[me:m, 0:k]  B[0:k, 0:n]        (mf rows of C)
//   n fringe:  C[0:me, ne:n] += alpha A[0:me, 0:k]  B[0:k, ne:n]       (nf columns of C)
// (the reference peels nothing: it zero-pads the quadrants, blocking.cpp:17-22; the
// paper's dynamic peeling, section 4.2, is the north-star's fringe handling).
// Through mm_kernel these ran whole 128 x 128 x 16 tile steps for a sliver of useful
// work (4097^3: a 1 x 4097 x 4097 update took 0.5 ms of 33 CTAs running the full k
// loop).  They are HBM-bound streaming problems: the long operand is read once.
//
// Deterministic: every output element is a fixed-order sum -- k-chunk partials are
// written to a workspace and added in ascending chunk order by thin_reduce_kernel; no
// atomics.  Element (i, j) of a view is p[i * rs + j * cs]; coalescing assumes the
// column-major layouts the engine hands over (rs == 1) and is merely slower otherwise.
#include "kernels.hpp"

namespace sb200 {
namespace {

constexpr int kThinMax = 16;     // fringe width limit (2^L - 1 <= 7 at L <= 3; up to 16 rows or
                                 // columns above a whole number of tiles, engine.cpp run_device)
constexpr int kChunkK = 256;     // k per partial chunk (m fringe: 16 x 256 doubles of shared memory)
constexpr int kChunkN = 64;      // k per partial chunk (n fringe: one thread per row of A, so
                                 // short chunks supply the CTAs that keep HBM busy)
constexpr int kRowThreads = 128;

// ---- n fringe: out[kc][j][i] = sum_{kk in chunk kc} A[i, kk] * B[kk, j], j < nf ------
// thread = one row i of the streamed operand A (M x K); B (K x nf) is broadcast
template <int NF>
__global__ void __launch_bounds__(kRowThreads)
    thin_n_kernel(const double* __restrict__ A, long long rs_a, long long cs_a,
                  const double* __restrict__ B, long long rs_b, long long cs_b, long M, long K,
                  double* __restrict__ part) {
    // rows padded to an even count: one 16-byte shared load per pair of columns
    constexpr int NP = (NF + 1) & ~1;
    __shared__ __align__(16) double Bs[kChunkN][NP];
    const long k0 = static_cast<long>(blockIdx.y) * kChunkN;
    const int kn = static_cast<int>(min(static_cast<long>(kChunkN), K - k0));
    for (int t = threadIdx.x; t < kn * NP; t += kRowThreads) {
        const int kk = t / NP, j = t % NP;
        Bs[kk][j] = j < NF ? B[(k0 + kk) * rs_b + j * cs_b] : 0.0;
    }
    __syncthreads();
    const long i = static_cast<long>(blockIdx.x) * kRowThreads + threadIdx.x;
    if (i >= M) return;
    double acc[NF];
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[j] = 0.0;
    const double* a = A + i * rs_a + k0 * cs_a;
    // eight loads of A in flight per thread (the kernel is bound by their latency:
    // ncu showed 0.14 eligible warps per scheduler with one load at a time)
    auto step = [&](int kk, double x) {
#pragma unroll
        for (int j2 = 0; j2 < NP / 2; ++j2) {
            const double2 bv = *reinterpret_cast<const double2*>(&Bs[kk][2 * j2]);
            acc[2 * j2] = fma(x, bv.x, acc[2 * j2]);
            if (2 * j2 + 1 < NF) acc[2 * j2 + 1] = fma(x, bv.y, acc[2 * j2 + 1]);
        }
    };
    int kk = 0;
    for (; kk + 8 <= kn; kk += 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __ldg(a + (kk + u) * cs_a);
#pragma unroll
        for (int u = 0; u < 8; ++u) step(kk + u, x[u]);
    }
    for (; kk < kn; ++kk) step(kk, __ldg(a + kk * cs_a));
#pragma unroll
    for (int j = 0; j < NF; ++j)
        part[(static_cast<long long>(blockIdx.y) * NF + j) * M + i] = acc[j];
}

// ---- m fringe: out[kc][i][j] = sum_{kk in chunk kc} A[i, kk] * B[kk, j], i < mf ------
// warp = one column j of the streamed operand B (K x N), lanes along k (contiguous for
// column-major B); the thin A (mf x K) chunk sits in shared memory
template <int MF>
__global__ void __launch_bounds__(256)
    thin_m_kernel(const double* __restrict__ A, long long rs_a, long long cs_a,
                  const double* __restrict__ B, long long rs_b, long long cs_b, long N, long K,
                  int cols_per_warp, double* __restrict__ part) {
    __shared__ double As[MF][kChunkK];
    const long k0 = static_cast<long>(blockIdx.y) * kChunkK;
    const int kn = static_cast<int>(min(static_cast<long>(kChunkK), K - k0));
    for (int t = threadIdx.x; t < kChunkK * MF; t += 256) {
        const int kk = t / MF, i = t % MF;
        As[i][kk] = kk < kn ? A[i * rs_a + (k0 + kk) * cs_a] : 0.0;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long j0 = (static_cast<long>(blockIdx.x) * 8 + warp) * cols_per_warp;
    for (long j = j0; j < min(N, j0 + cols_per_warp); ++j) {
        double acc[MF];
#pragma unroll
        for (int i = 0; i < MF; ++i) acc[i] = 0.0;
        const double* b = B + k0 * rs_b + j * cs_b;
        // four loads of B in flight per lane (latency-bound otherwise, as thin_n_kernel)
        int kk = lane;
        for (; kk + 96 < kn; kk += 128) {
            double x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = __ldg(b + (kk + 32 * u) * rs_b);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < MF; ++i) acc[i] = fma(As[i][kk + 32 * u], x[u], acc[i]);
        }
        for (; kk < kn; kk += 32) {
            const double x = __ldg(b + kk * rs_b);
#pragma unroll
            for (int i = 0; i < MF; ++i) acc[i] = fma(As[i][kk], x, acc[i]);
        }
        // fixed butterfly: the same order on every run
#pragma unroll
        for (int i = 0; i < MF; ++i) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
                acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
        }
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < MF; ++i)
                part[(static_cast<long long>(blockIdx.y) * MF + i) * N + j] = acc[i];
        }
    }
}

// ---- chunk partials into C: C[l, t] += alpha * sum_kc part[kc][t][l] (ascending kc) ----
// l runs over the long dimension (stride sl in C), t over the thin one (stride st)
__global__ void __launch_bounds__(256)
    thin_reduce_kernel(const double* __restrict__ part, int nkc, int thin, long len, double alpha,
                       double* __restrict__ C, long long sl, long long st) {
    const long l = static_cast<long>(blockIdx.x) * 256 + threadIdx.x;
    const int t = blockIdx.y;
    if (l >= len) return;
    double s = 0.0;
    for (int kc = 0; kc < nkc; ++kc) s += part[(static_cast<long long>(kc) * thin + t) * len + l];
    double* c = C + l * sl + t * st;
    *c = fma(alpha, s, *c);
}

// ---- k fringe: C[i, j] += alpha * sum_{kk < kf} A[i, kk] * B[kk, j] -------------------
// thread = one row i, a strip of kColsPerBlock columns per block
constexpr int kColsPerBlock = 16;
template <int KF>
__global__ void __launch_bounds__(kRowThreads)
    rank_kf_kernel(const double* __restrict__ A, long long rs_a, long long cs_a,
                   const double* __restrict__ B, long long rs_b, long long cs_b,
                   double* __restrict__ C, long long rs_c, long long cs_c, long M, long N,
                   double alpha) {
    __shared__ double Bs[KF][kColsPerBlock];
    const long j0 = static_cast<long>(blockIdx.y) * kColsPerBlock;
    const int jn = static_cast<int>(min(static_cast<long>(kColsPerBlock), N - j0));
    for (int t = threadIdx.x; t < KF * kColsPerBlock; t += kRowThreads) {
        const int kk = t / kColsPerBlock, j = t % kColsPerBlock;
        Bs[kk][j] = j < jn ? B[kk * rs_b + (j0 + j) * cs_b] : 0.0;
    }
    __syncthreads();
    const long i = static_cast<long>(blockIdx.x) * kRowThreads + threadIdx.x;
    if (i >= M) return;
    double a[KF];
#pragma unroll
    for (int kk = 0; kk < KF; ++kk) a[kk] = __ldg(A + i * rs_a + kk * cs_a);
    for (int j = 0; j < jn; ++j) {
        double s = 0.0;
#pragma unroll
        for (int kk = 0; kk < KF; ++kk) s = fma(a[kk], Bs[kk][j], s);
        double* c = C + i * rs_c + (j0 + j) * cs_c;
        *c = fma(alpha, s, *c);
    }
}

template <int W>
cudaError_t thin_n_w(const double* A, long long rs_a, long long cs_a, const double* B,
                     long long rs_b, long long cs_b, long M, long K, double* part, dim3 grid,
                     cudaStream_t s) {
    thin_n_kernel<W><<<grid, kRowThreads, 0, s>>>(A, rs_a, cs_a, B, rs_b, cs_b, M, K, part);
    return cudaGetLastError();
}
template <int W>
cudaError_t thin_m_w(const double* A, long long rs_a, long long cs_a, const double* B,
                     long long rs_b, long long cs_b, long N, long K, int cpw, double* part,
                     dim3 grid, cudaStream_t s) {
    thin_m_kernel<W><<<grid, 256, 0, s>>>(A, rs_a, cs_a, B, rs_b, cs_b, N, K, cpw, part);
    return cudaGetLastError();
}
template <int W>
cudaError_t rank_w(const double* A, long long rs_a, long long cs_a, const double* B,
                   long long rs_b, long long cs_b, double* C, long long rs_c, long long cs_c,
                   long M, long N, double alpha, dim3 grid, cudaStream_t s) {
    rank_kf_kernel<W><<<grid, kRowThreads, 0, s>>>(A, rs_a, cs_a, B, rs_b, cs_b, C, rs_c, cs_c, M,
                                                   N, alpha);
    return cudaGetLastError();
}

#define SB200_WIDTH_SWITCH(w, CALL)                                                     \
    switch (w) {                                                                        \
        case 1: return CALL(1);                                                         \
        case 2: return CALL(2);                                                         \
        case 3: return CALL(3);                                                         \
        case 4: return CALL(4);                                                         \
        case 5: return CALL(5);                                                         \
        case 6: return CALL(6);                                                         \
        case 7: return CALL(7);                                                         \
        case 8: return CALL(8);                                                         \
        case 9: return CALL(9);                                                         \
        case 10: return CALL(10);                                                       \
        case 11: return CALL(11);                                                       \
        case 12: return CALL(12);                                                       \
        case 13: return CALL(13);                                                       \
        case 14: return CALL(14);                                                       \
        case 15: return CALL(15);                                                       \
        case 16: return CALL(16);                                                       \
        default: return cudaErrorInvalidValue;                                          \
    }

}  // namespace

int fringe_max_width() { return kThinMax; }

size_t fringe_partial_bytes(long long_len, int thin, long K) {
    const long nkc = (K + kChunkN - 1) / kChunkN;  // (the finer of the two chunkings)
    return static_cast<size_t>(nkc) * static_cast<size_t>(thin) * static_cast<size_t>(long_len) * 8;
}

// part[kc][j][i] = sum over k-chunk kc of A (M x K) * B (K x nf), nf <= 8;
// part: fringe_partial_bytes(M, nf, K); returns the chunk count in *nkc_out
cudaError_t launch_fringe_n(const double* A, long long rs_a, long long cs_a, const double* B,
                            long long rs_b, long long cs_b, long M, int nf, long K, double* part,
                            int* nkc_out, cudaStream_t s) {
    const int nkc = static_cast<int>((K + kChunkN - 1) / kChunkN);
    *nkc_out = nkc;
    const dim3 grid(static_cast<unsigned>((M + kRowThreads - 1) / kRowThreads),
                    static_cast<unsigned>(nkc));
#define CALL(W) thin_n_w<W>(A, rs_a, cs_a, B, rs_b, cs_b, M, K, part, grid, s)
    SB200_WIDTH_SWITCH(nf, CALL)
#undef CALL
}

// part[kc][i][j] = sum over k-chunk kc of A (mf x K) * B (K x N), mf <= 8;
// part: fringe_partial_bytes(N, mf, K)
cudaError_t launch_fringe_m(const double* A, long long rs_a, long long cs_a, const double* B,
                            long long rs_b, long long cs_b, int mf, long N, long K, double* part,
                            int* nkc_out, cudaStream_t s) {
    const int nkc = static_cast<int>((K + kChunkK - 1) / kChunkK);
    *nkc_out = nkc;
    const int cpw = 4;  // columns per warp: 32 per block
    const dim3 grid(static_cast<unsigned>((N + 8 * cpw - 1) / (8 * cpw)), static_cast<unsigned>(nkc));
#define CALL(W) thin_m_w<W>(A, rs_a, cs_a, B, rs_b, cs_b, N, K, cpw, part, grid, s)
    SB200_WIDTH_SWITCH(mf, CALL)
#undef CALL
}

// C[l, t] += alpha * sum_kc part[kc][t][l], kc ascending; l < len along stride sl of C,
// t < thin along stride st
cudaError_t launch_fringe_reduce(const double* part, int nkc, int thin, long len, double alpha,
                                 double* C, long long sl, long long st, cudaStream_t s) {
    const dim3 rgrid(static_cast<unsigned>((len + 255) / 256), static_cast<unsigned>(thin));
    thin_reduce_kernel<<<rgrid, 256, 0, s>>>(part, nkc, thin, len, alpha, C, sl, st);
    return cudaGetLastError();
}

// C (M x N) += alpha * A (M x kf) * B (kf x N), kf <= 8
cudaError_t launch_fringe_k(const double* A, long long rs_a, long long cs_a, const double* B,
                            long long rs_b, long long cs_b, double* C, long long rs_c,
                            long long cs_c, long M, long N, int kf, double alpha, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((M + kRowThreads - 1) / kRowThreads),
                    static_cast<unsigned>((N + kColsPerBlock - 1) / kColsPerBlock));
#define CALL(W) rank_w<W>(A, rs_a, cs_a, B, rs_b, cs_b, C, rs_c, cs_c, M, N, alpha, grid, s)
    SB200_WIDTH_SWITCH(kf, CALL)
#undef CALL
}

}  // namespace sb200
