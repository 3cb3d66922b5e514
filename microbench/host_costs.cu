// Host-side cost of the CUDA calls one strassen_gemm_device call makes (tensor-map
// encodes, pointer queries, events, small memsets, kernel launches with the ~24 KB
// MMParams block vs a small one), microseconds per call.
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

struct Big { CUtensorMap m[176]; int x; };   // ~22.5 KB, like MMParams
struct Small { CUtensorMap m[4]; int x; };
__global__ void kbig(const __grid_constant__ Big p) { if (p.x == 12345) printf("x"); }
__global__ void ksmall(const __grid_constant__ Small p) { if (p.x == 12345) printf("x"); }

template <class F> double us(F f, int n = 2000) {
    f();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

int main() {
    double* d;
    cudaMalloc(&d, 1 << 26);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
    CUtensorMap map;
    cuuint64_t dims[2] = {1024, 1024}, strides[1] = {8192};
    cuuint32_t box[2] = {16, 16}, es[2] = {1, 1};
    printf("cuTensorMapEncodeTiled: %.2f us\n", us([&] {
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }));
    cudaPointerAttributes a;
    printf("cudaPointerGetAttributes: %.2f us\n", us([&] { cudaPointerGetAttributes(&a, d); }));
    printf("cudaEventRecord + cudaStreamWaitEvent: %.2f us\n",
           us([&] { cudaEventRecord(ev, s); cudaStreamWaitEvent(s, ev, 0); }));
    printf("cudaMemsetAsync (4 KB): %.2f us\n", us([&] { cudaMemsetAsync(d, 0, 4096, s); }));
    static Big big{};
    static Small small{};
    printf("launch, 22.5 KB params: %.2f us\n", us([&] { kbig<<<148, 384, 0, s>>>(big); }));
    printf("launch, 0.5 KB params: %.2f us\n", us([&] { ksmall<<<148, 384, 0, s>>>(small); }));
    cudaStreamSynchronize(s);
    printf("memcpy of 22.5 KB struct (host): %.3f us\n", us([&] { static Big b2; b2 = big; }));
    return 0;
}
