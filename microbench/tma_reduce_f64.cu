// Probe: does cp.reduce.async.bulk.tensor (.add) accept an FP64 tensor map on
// sm_100a?  Adds a 16 x 128 box staged in shared memory (128-byte swizzle)
// into a column-major 256 x 256 fp64 matrix and checks the result.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap map, int r0, int c0) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s = sm + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(sm)) & 1023u)) & 1023u);
    // box {16 rows, 128 cols}: col c at c*128, row r chunk ((r/2) ^ (c%8)), +8*(r%2)
    for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) {
        const int r = i % 16, c = i / 16;
        double v = 1000.0 * c + r;  // distinct per element
        *reinterpret_cast<double*>(s + c * 128 + (((r / 2) ^ (c % 8)) << 4) + (r % 2) * 8) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s));
        asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];"
                     ::"l"(reinterpret_cast<uint64_t>(&map)), "r"(r0), "r"(c0), "r"(sa) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// Finding: rows (the inner dimension) clip at 16-byte granularity -- with an odd
// row count the element after the last row is written too -- while columns clip
// exactly.  The Strassen epilogue therefore uses the reduce-add only where a
// tile does not end inside a quadrant with an odd row count.
int run(int dim_rows, int dim_cols, int r0, int c0);
int main() {
    int bad = run(256, 256, 32, 64);
    bad += run(250, 256, 240, 64);   // rows 250..255 of the box outside the map: stay 1.0
    bad += run(256, 100, 32, 64);    // columns 100..191 outside the map
    const int odd = run(37, 256, 32, 64);  // expected to fail: row 37 is written
    printf("odd row count clipped exactly: %s\n", odd ? "no" : "yes");
    return bad != 0;
}

int run(int dim_rows, int dim_cols, int r0, int c0) {
    const int n = 256;
    std::vector<double> h(n * n, 1.0);
    double* d;
    cudaMalloc(&d, n * n * 8);
    cudaMemcpy(d, h.data(), n * n * 8, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(dim_rows), static_cast<cuuint64_t>(dim_cols)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(n) * 8};
    cuuint32_t box[2] = {16, 128}, es[2] = {1, 1};
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", static_cast<int>(r));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    k<<<1, 128, 20000>>>(map, r0, c0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    cudaMemcpy(h.data(), d, n * n * 8, cudaMemcpyDeviceToHost);
    long bad = 0, touched = 0;
    for (int c = 0; c < n; ++c)
        for (int rr = 0; rr < n; ++rr) {
            double want = 1.0;
            if (rr >= r0 && rr < r0 + 16 && rr < dim_rows && c >= c0 && c < c0 + 128 && c < dim_cols) { want += 1000.0 * (c - c0) + (rr - r0); ++touched; }
            if (h[rr + c * n] != want) ++bad;
        }
    printf("dims %dx%d box at (%d,%d): touched %ld bad %ld\n", dim_rows, dim_cols, r0, c0, touched, bad);
    cudaFree(d);
    return bad != 0;
}
