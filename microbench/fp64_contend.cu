// DADD throughput of "side" warps while 8 warps saturate the DMMA pipe, and an
// integer-pipe exact fp64 add as the alternative.  Per-role completion times
// are measured with clock64 inside the kernel (DMMA warps run a fixed amount
// of work; side warps run D adds).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// Exact IEEE-754 binary64 addition (round to nearest even) on the integer
// pipes.  Fast path for finite normal operands; anything else falls back to
// the hardware DADD (rare in practice).
__device__ __forceinline__ double iadd_f64(double x, double y) {
  uint64_t a = __double_as_longlong(x), b = __double_as_longlong(y);
  uint32_t ea = (uint32_t)(a >> 52) & 0x7ff, eb = (uint32_t)(b >> 52) & 0x7ff;
  if (ea - 1u >= 0x7feu || eb - 1u >= 0x7feu) return x + y;
  uint64_t aa = a & 0x7fffffffffffffffull, bb = b & 0x7fffffffffffffffull;
  if (bb > aa) { uint64_t t = a; a = b; b = t; uint32_t te = ea; ea = eb; eb = te; }
  const uint64_t sign = a & 0x8000000000000000ull;
  const bool sub = ((a ^ b) >> 63) != 0;
  uint64_t ma = ((a & 0xfffffffffffffull) | 0x10000000000000ull) << 10;  // bit 62 leading
  uint64_t mb = ((b & 0xfffffffffffffull) | 0x10000000000000ull) << 10;
  uint32_t d = ea - eb;
  if (d >= 63) mb = 1;  // sticky only
  else if (d) { uint64_t st = (mb << (64 - d)) != 0; mb = (mb >> d) | st; }
  int e = (int)ea;
  uint64_t m;
  if (!sub) {
    m = ma + mb;
    if (m >> 63) { m = (m >> 1) | (m & 1); e += 1; }
  } else {
    m = ma - mb;
    if (m == 0) return 0.0;
    int lz = __clzll(m) - 1;
    m <<= lz; e -= lz;
    if (e <= 0) return x + y;  // subnormal result: hardware
  }
  uint64_t rb = m & 0x3ff; m >>= 10;
  if (rb > 0x200 || (rb == 0x200 && (m & 1))) { m += 1; if (m >> 53) { m >>= 1; e += 1; } }
  if (e >= 0x7ff) return x + y;  // overflow: hardware
  return __longlong_as_double((long long)(sign | ((uint64_t)e << 52) | (m & 0xfffffffffffffull)));
}

template <int MODE, int ILP>  // MODE 0: DADD side warps, 1: integer add side warps
__global__ void k_contend(unsigned long long* t_out, double* sink, int dmma_iters, int side_iters,
                          int side_warps) {
  const int warp = threadIdx.x / 32;
  unsigned long long t0 = clock64();
  double s = 0;
  if (warp < 8) {
    double c[16][2];
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j][0] = c[j][1] = 0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int i = 0; i < dmma_iters; ++i) {
#pragma unroll
      for (int g = 0; g < 32; ++g) dmma(c[g % 16][0], c[g % 16][1], a, b);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) s += c[j][0] + c[j][1];
  } else if (warp < 8 + side_warps) {
    double y[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) y[j] = 1.0 + threadIdx.x + j;
    const double a = 1.0 + threadIdx.x * 1e-3;
    for (int i = 0; i < side_iters; ++i) {
#pragma unroll
      for (int j = 0; j < ILP; ++j) {
        if (MODE == 0) asm volatile("add.f64 %0, %0, %1;" : "+d"(y[j]) : "d"(a));
        else y[j] = iadd_f64(y[j], a);
      }
    }
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += y[j];
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x % 32 == 0 && blockIdx.x == 0) t_out[warp] = t1 - t0;
  if (s == 12345.678) sink[blockIdx.x] = s;
}

__global__ void k_check(double* out, const double* x, const double* y, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = iadd_f64(x[i], y[i]);
}

template <int MODE, int ILP>
void run(unsigned long long* dt, double* sink, int sms, int side_warps, int dmma_iters, int side_iters,
         const char* name) {
  k_contend<MODE, ILP><<<sms, 512>>>(dt, sink, dmma_iters, side_iters, side_warps);
  cudaDeviceSynchronize();
  unsigned long long h[16];
  cudaMemcpy(h, dt, sizeof(h), cudaMemcpyDeviceToHost);
  double dm = 0, sd = 0;
  for (int w = 0; w < 8; ++w) dm += h[w];
  for (int w = 8; w < 8 + side_warps; ++w) sd += h[w];
  dm /= 8; sd /= (side_warps ? side_warps : 1);
  double dmma_per_smsp = 2.0 * 32 * dmma_iters;  // 2 DMMA warps per SMSP
  double adds_per_warp = (double)ILP * side_iters;
  printf("%-34s side=%2d ILP=%2d: DMMA warps %9.0f clk (%.2f clk/DMMA/SMSP); side warps %9.0f clk "
         "(%.1f clk per warp-add)\n", name, side_warps, ILP, dm, dm / dmma_per_smsp, sd,
         side_warps ? sd / adds_per_warp : 0.0);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  unsigned long long* dt; cudaMalloc(&dt, 16 * 8);
  double* sink; cudaMalloc(&sink, 1 << 20);
  // alone
  run<0, 8>(dt, sink, sms, 0, 2000, 0, "DMMA only");
  run<0, 8>(dt, sink, sms, 4, 0, 20000, "DADD only (no DMMA)");
  run<1, 8>(dt, sink, sms, 4, 0, 4000, "intadd only (no DMMA)");
  run<1, 8>(dt, sink, sms, 8, 0, 4000, "intadd only (no DMMA)");
  // contended: DMMA warps run long; side warps fixed work
  run<0, 8>(dt, sink, sms, 4, 4000, 2000, "DADD under DMMA");
  run<0, 16>(dt, sink, sms, 4, 4000, 1000, "DADD under DMMA");
  run<0, 8>(dt, sink, sms, 8, 4000, 2000, "DADD under DMMA");
  run<1, 8>(dt, sink, sms, 4, 4000, 1000, "intadd under DMMA");
  run<1, 8>(dt, sink, sms, 8, 4000, 1000, "intadd under DMMA");
  // correctness of iadd_f64 vs hardware on random / edge inputs
  const int n = 1 << 22;
  double *hx = new double[n], *hy = new double[n], *hr = new double[n];
  uint64_t s = 88172645463325252ull;
  auto rnd = [&] { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
  for (int i = 0; i < n; ++i) {
    uint64_t bx = rnd(), by = rnd();
    int mode = i % 8;
    if (mode < 4) {  // random doubles of moderate exponent
      hx[i] = ((double)(int64_t)(bx >> 11) / 9007199254740992.0) * (mode == 0 ? 1 : (double)(1ll << (bx % 40)));
      hy[i] = ((double)(int64_t)(by >> 11) / 9007199254740992.0) * (mode == 1 ? -1.0 : 1.0) * ((by % 7) ? 1.0 : 1e-300);
      if (mode == 3) hy[i] = -hx[i] * (1.0 + ((double)(by % 1000)) * 1e-16);
    } else {  // raw bit patterns (incl. inf/nan/subnormal)
      memcpy(&hx[i], &bx, 8);
      uint64_t b2 = (mode == 5) ? (bx ^ 0x8000000000000000ull) + (by % 3) : by;
      memcpy(&hy[i], &b2, 8);
    }
  }
  double *dx, *dy, *dr;
  cudaMalloc(&dx, n * 8); cudaMalloc(&dy, n * 8); cudaMalloc(&dr, n * 8);
  cudaMemcpy(dx, hx, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, hy, n * 8, cudaMemcpyHostToDevice);
  k_check<<<(n + 255) / 256, 256>>>(dr, dx, dy, n);
  cudaMemcpy(hr, dr, n * 8, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < n; ++i) {
    double want = hx[i] + hy[i];
    uint64_t w, g;
    memcpy(&w, &want, 8); memcpy(&g, &hr[i], 8);
    bool both_nan = (want != want) && (hr[i] != hr[i]);
    if (w != g && !both_nan) { if (bad < 5) printf("mismatch %a + %a = %a got %a\n", hx[i], hy[i], want, hr[i]); ++bad; }
  }
  printf("iadd_f64 bitwise check: %ld mismatches of %d\n", bad, n);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
