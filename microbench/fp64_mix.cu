// How DADD interleaving granularity affects DMMA throughput on sm_100a.
// Each warp loops: G independent DMMA.8, then D independent DADDs.
// Also: DMMA-only warps co-resident with DADD-only warps on the same SMSP.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int G, int D>
__global__ void k_mix(double* out, int iters) {
  double c[16][2];
  double y[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) { c[j][0] = c[j][1] = 0; y[j] = threadIdx.x + j; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int g = 0; g < G; ++g) dmma(c[g % 16][0], c[g % 16][1], a, b);
#pragma unroll
    for (int d = 0; d < D; ++d) asm volatile("add.f64 %0, %0, %1;" : "+d"(y[d % 16]) : "d"(a));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += c[j][0] + c[j][1] + y[j];
  if (s == 12345.678) out[blockIdx.x] = s;
}

// warps 0..7: DMMA only; warps 8..11: DADD only at a fixed rate (D per G-DMMA-time)
template <int D>
__global__ void k_split(double* out, int iters) {
  const int warp = threadIdx.x / 32;
  double s = 0;
  if (warp < 8) {
    double c[16][2];
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j][0] = c[j][1] = 0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int g = 0; g < 32; ++g) dmma(c[g % 16][0], c[g % 16][1], a, b);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) s += c[j][0] + c[j][1];
  } else {
    double y[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) y[j] = threadIdx.x + j;
    double a = 1.0 + threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int d = 0; d < D; ++d) asm volatile("add.f64 %0, %0, %1;" : "+d"(y[d % 16]) : "d"(a));
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) s += y[j];
  }
  if (s == 12345.678) out[blockIdx.x] = s;
}

template <typename F>
float time_it(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); launch();
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 3;
}

template <int G, int D>
void run(double* out, int sms) {
  const int iters = 65536 / G;
  float ms = time_it([&] { k_mix<G, D><<<sms, 256>>>(out, iters); });
  double fl = 2.0 * 256 * G * iters * 8.0 * sms;
  printf("mix G=%3d D=%3d (DADD per DMMA %.3f): DMMA %.2f TF/s\n", G, D, (double)D / G, fl / ms / 1e9);
}

template <int D>
void run_split(double* out, int sms) {
  const int iters = 2048;
  float ms = time_it([&] { k_split<D><<<sms, 384>>>(out, iters); });
  double fl = 2.0 * 256 * 32 * iters * 8.0 * sms;
  printf("split 8 DMMA warps + 4 DADD warps, D=%3d per loop: DMMA %.2f TF/s\n", D, fl / ms / 1e9);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 1 << 20);
  int sms = p.multiProcessorCount;
  run<32, 0>(out, sms);
  run<8, 1>(out, sms);
  run<32, 1>(out, sms);
  run<32, 2>(out, sms);
  run<32, 4>(out, sms);
  run<64, 8>(out, sms);
  run<128, 16>(out, sms);
  run<256, 32>(out, sms);
  run<128, 4>(out, sms);
  run<256, 8>(out, sms);
  run_split<0>(out, sms);
  run_split<1>(out, sms);
  run_split<2>(out, sms);
  run_split<4>(out, sms);
  run_split<8>(out, sms);
  run_split<16>(out, sms);
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
