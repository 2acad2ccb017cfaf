// How fast does one SM receive a 96 KB token operand from L2?  (small-model
// row GEMM question: a [64 tokens][768] bf16 operand per CTA)
//
//   mode 0: 12 tensor-TMA loads, boxes {64 cols, 64 rows}, 128B swizzle
//   mode 1: one cp.async.bulk of 96 KB (a pre-swizzled global image)
//   mode 2: 12 cp.async.bulk of 8 KB
//   mode 3: 24 tensor-TMA loads, boxes {64 cols, 32 rows}
//
// Each CTA repeats the load `reps` times (waiting for each), timing with
// %globaltimer; the buffer is L2-resident after the first pass.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_vs_bulk tma_vs_bulk.cu -lcuda && ./tma_vs_bulk
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(s32(bar)),
        "r"(parity)
        : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap m64, const __grid_constant__ CUtensorMap m32, const uint8_t* img,
                  int mode, int reps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    uint8_t* buf = sm + ((1024u - (s32(sm) & 1023u)) & 1023u);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t_sum = 0;
    for (int r = 0; r < reps; ++r) {
        if (threadIdx.x == 0) {
            const uint64_t t0 = gtime();
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(96 * 1024));
            if (mode == 0 || mode == 3) {
                const int rows = mode == 0 ? 64 : 32;
                const CUtensorMap* m = mode == 0 ? &m64 : &m32;
                for (int kb = 0; kb < 12; ++kb)
                    for (int t0r = 0; t0r < 64; t0r += rows)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                                s32(buf + kb * 8192 + t0r * 128)),
                            "l"(m), "r"(kb * 64), "r"(t0r), "r"(s32(&bar))
                            : "memory");
            } else {
                const int n = mode == 1 ? 1 : 12, bytes = 96 * 1024 / n;
                for (int i = 0; i < n; ++i)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            s32(buf + i * bytes)),
                        "l"(img + (size_t)i * bytes), "r"(bytes), "r"(s32(&bar))
                        : "memory");
            }
            mbar_wait(&bar, r & 1);
            if (r > 0) t_sum += gtime() - t0;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = t_sum / (reps - 1);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int T = 64, K = 768;
    void* x;
    cudaMalloc(&x, (size_t)T * K * 2);
    cudaMemset(x, 0, (size_t)T * K * 2);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fn;
    CUtensorMap m64, m32;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)T}, strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box64[2] = {64, 64}, box32[2] = {64, 32}, es[2] = {1, 1};
    enc(&m64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&m32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    unsigned long long* out;
    cudaMalloc(&out, 148 * sizeof(unsigned long long));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const char* names[4] = {"tensor TMA 12 x {64,64}", "bulk 1 x 96 KB", "bulk 12 x 8 KB", "tensor TMA 24 x {64,32}"};
    for (int grid : {1, 12, 48, 148})
        for (int mode = 0; mode < 4; ++mode) {
            k<<<grid, 128, 100 * 1024>>>(m64, m32, (const uint8_t*)x, mode, 20, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            std::vector<unsigned long long> h(grid);
            cudaMemcpy(h.data(), out, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
            unsigned long long mx = 0, sum = 0;
            for (auto v : h) {
                mx = std::max(mx, v);
                sum += v;
            }
            printf("grid %3d  %-26s  mean %6.0f ns  max %6llu ns  (%.0f GB/s per SM)\n", grid, names[mode],
                   (double)sum / grid, mx, 96.0 * 1024 / ((double)sum / grid));
        }
    return 0;
}
