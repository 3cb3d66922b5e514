// FP64 pipe microbenchmark for sm_100a: DFMA (FMA pipe) vs DMMA (mma.sync f64)
// and whether DADD co-issues with DMMA.  Establishes the FP64 peak used as the
// roofline denominator (MEASURED_PEAKS.json has only bf16/HBM).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[blockIdx.x] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NACC, int NADD>
__global__ void k_dmma(double* out, int iters, double a0, double b0) {
  double c[NACC][2];
  double y[NADD > 0 ? NADD : 1];
#pragma unroll
  for (int j = 0; j < NACC; ++j) { c[j][0] = 0; c[j][1] = 0; }
#pragma unroll
  for (int j = 0; j < (NADD > 0 ? NADD : 1); ++j) y[j] = threadIdx.x + j;
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) dmma(c[j][0], c[j][1], a, b);
#pragma unroll
    for (int j = 0; j < NADD; ++j) y[j] = y[j] + a;
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1];
#pragma unroll
  for (int j = 0; j < (NADD > 0 ? NADD : 1); ++j) s += y[j];
  if (s == 12345.678) out[blockIdx.x] = s;
}

template <typename F>
float time_it(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();  // warm
  launch();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d clock(kHz) %d\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  const int sms = p.multiProcessorCount;
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256, blocks = sms * bpsm, iters = 20000;
    float ms = time_it([&] { k_dfma<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); }, 5);
    double fl = 2.0 * 32 * iters * (double)threads * blocks;
    printf("DFMA   blocks/SM=%d: %.3f ms  %.2f TFLOP/s\n", bpsm, ms, fl / ms / 1e9);
  }
  CK(cudaGetLastError());
  for (int bpsm : {1, 2, 4}) {
    int threads = 256, blocks = sms * bpsm, iters = 4000;
    float ms = time_it([&] { k_dmma<8, 0><<<blocks, threads>>>(out, iters, 1.0, 1.0); }, 5);
    double fl = 2.0 * 256 * 8 * iters * (double)(threads / 32) * blocks;
    printf("DMMA8  acc=8 blocks/SM=%d: %.3f ms  %.2f TFLOP/s\n", bpsm, ms, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2}) {
    int threads = 256, blocks = sms * bpsm, iters = 4000;
    float ms = time_it([&] { k_dmma<16, 0><<<blocks, threads>>>(out, iters, 1.0, 1.0); }, 5);
    double fl = 2.0 * 256 * 16 * iters * (double)(threads / 32) * blocks;
    printf("DMMA8  acc=16 blocks/SM=%d: %.3f ms  %.2f TFLOP/s\n", bpsm, ms, fl / ms / 1e9);
  }
  {
    int threads = 256, blocks = sms * 2, iters = 4000;
    float ms = time_it([&] { k_dmma<8, 8><<<blocks, threads>>>(out, iters, 1.0, 1.0); }, 5);
    double fl = 2.0 * 256 * 8 * iters * (double)(threads / 32) * blocks;
    printf("DMMA8+8DADD blocks/SM=2: %.3f ms  mma %.2f TFLOP/s\n", ms, fl / ms / 1e9);
    ms = time_it([&] { k_dmma<8, 32><<<blocks, threads>>>(out, iters, 1.0, 1.0); }, 5);
    printf("DMMA8+32DADD blocks/SM=2: %.3f ms  mma %.2f TFLOP/s\n", ms, fl / ms / 1e9);
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
