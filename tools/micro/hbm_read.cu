// Read-only HBM streaming ceiling on this B200: what a weight / KV streaming
// kernel can reach at best, next to the copy (read + write) peak that
// MEASURED_PEAKS.json holds.  Three variants over a 4 GiB buffer:
//   ldg     : 148*k CTAs x 512 threads, 128-bit ld.global.nc, 8 loads in flight per thread
//   bulk    : one CTA per SM, cp.async.bulk (1-D TMA) 32 KB stages into an mbarrier
//             ring of S stages (the mechanism of k_gemm / k_attention_tcp)
//   bulk2   : the same with 2 CTAs per SM (half the ring each)
// Timed with CUDA events, best of 10.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_read hbm_read.cu && ./hbm_read
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_ldg(const int4* __restrict__ p, size_t n, int* out) {
    int acc = 0;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                                                 : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                                                 : "l"(p + i + u * stride));
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678) *out = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const char* __restrict__ p, size_t bytes, int stages, int* out) {
    extern __shared__ __align__(128) char smem[];
    constexpr int kStage = 32768;
    uint64_t* full = (uint64_t*)(smem + stages * kStage);
    uint64_t* empty = full + 8;
    const size_t per = (bytes / gridDim.x) & ~(size_t)(kStage - 1);
    const char* base = p + (size_t)blockIdx.x * per;
    const int nst = (int)(per / kStage);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared.b64 [%0], 4;" ::"r"(su32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (int i = 0; i < nst; ++i) {
                int s = i % stages;
                uint32_t ph = ((i / stages) & 1) ^ 1;
                asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" ::"r"(
                                 su32(&empty[s])), "r"(ph));
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(kStage));
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                        su32(smem + s * kStage)),
                    "l"(base + (size_t)i * kStage), "r"(kStage), "r"(su32(&full[s])), "l"(pol)
                    : "memory");
            }
        }
    } else if (warp <= 4) {  // 4 consumer warps touch one word per stage and release it
        int acc = 0;
        for (int i = 0; i < nst; ++i) {
            int s = i % stages;
            uint32_t ph = (i / stages) & 1;
            asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" ::"r"(
                             su32(&full[s])), "r"(ph));
            acc ^= ((int*)(smem + s * kStage))[(warp - 1) * 32 + lane];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&empty[s])));
        }
        if (acc == 0x12345678) *out = acc;
    }
}

// k_gemm's weight stream: 2-D TMA boxes of 64 columns x 256 rows (SW128) of a
// row-major [rows][K] bf16 matrix, units (tile, k-block) tile-major, split
// stream-K over the CTAs -- each box touches 256 rows x 128 B
__global__ void k_tma2d(const __grid_constant__ CUtensorMap tm, long long tiles, int KB, int stages, int* out) {
    extern __shared__ __align__(1024) char smem2[];
    char* smem = smem2;
    constexpr int kStage = 32768;
    uint64_t* full = (uint64_t*)(smem + stages * kStage);
    uint64_t* empty = full + 8;
    const long long U = tiles * KB, G = gridDim.x;
    const long long u0 = blockIdx.x * U / G, u1 = (blockIdx.x + 1) * U / G;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared.b64 [%0], 4;" ::"r"(su32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (long long u = u0; u < u1; ++u) {
                int i = (int)(u - u0), s = i % stages;
                uint32_t ph = ((i / stages) & 1) ^ 1;
                asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" ::"r"(
                                 su32(&empty[s])), "r"(ph));
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(kStage));
                int x = (int)(u % KB) * 64, y = (int)(u / KB) * 256;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                    " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(smem + s * kStage)),
                    "l"(&tm), "r"(x), "r"(y), "r"(su32(&full[s])), "l"(pol)
                    : "memory");
            }
        }
    } else if (warp <= 4) {
        int acc = 0;
        for (long long u = u0; u < u1; ++u) {
            int i = (int)(u - u0), s = i % stages;
            uint32_t ph = (i / stages) & 1;
            asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" ::"r"(
                             su32(&full[s])), "r"(ph));
            acc ^= ((int*)(smem + s * kStage))[(warp - 1) * 32 + lane];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&empty[s])));
        }
        if (acc == 0x12345678) *out = acc;
    }
}

// k_gemm's two operand streams without the MMA: the weight box (64 x 256,
// HBM) plus a token box (64 x T, an L2-resident [T][K] matrix) per unit, the
// token ring TS deep.  With a cluster of C CTAs (C > 1) the CTAs walk the same
// k-blocks of C adjacent tiles in lockstep and the token box is multicast:
// CTA r loads rows [r T/C, (r+1) T/C) into every CTA of the cluster; a token
// stage is refilled once all C CTAs released it (remote mbarrier arrives).
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t ph) {
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" ::"r"(bar), "r"(ph));
}
__global__ void k_wtok(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
                       long long tiles, int KB, int T, int stages, int tstages, int* out) {
    extern __shared__ __align__(1024) char smem3[];
    char* smem = smem3;
    constexpr int kStage = 32768;
    uint32_t C;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(C));
    const uint32_t rank = C > 1 ? cluster_rank() : 0;
    const int tbytes = T * 128;
    char* tring = smem + stages * kStage;
    uint64_t* full = (uint64_t*)(tring + tstages * tbytes);
    uint64_t* empty = full + 8;
    uint64_t* tfull = empty + 8;
    uint64_t* tempty = tfull + 8;
    const long long Uc = tiles / C * KB, G = gridDim.x / C, cid = blockIdx.x / C;
    const long long u0 = cid * Uc / G, u1 = (cid + 1) * Uc / G;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&empty[s])));
        }
        for (int s = 0; s < tstages; ++s) {
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&tfull[s])));
            asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(&tempty[s])), "r"(C));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (C > 1) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    else __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (warp == 0 && lane == 0) {  // weights
        for (long long u = u0; u < u1; ++u) {
            int i = (int)(u - u0), s = i % stages;
            wait_parity(su32(&empty[s]), ((i / stages) & 1) ^ 1);
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(kStage));
            int x = (int)(u % KB) * 64, y = (int)((u / KB) * C + rank) * 256;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(smem + s * kStage)),
                "l"(&tw), "r"(x), "r"(y), "r"(su32(&full[s])), "l"(pol)
                : "memory");
        }
    } else if (warp == 1 && lane == 0) {  // tokens
        uint64_t keep;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
        const int rows = T / (int)C;
        for (long long u = u0; u < u1; ++u) {
            int i = (int)(u - u0), s = i % tstages;
            wait_parity(su32(&tempty[s]), ((i / tstages) & 1) ^ 1);
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&tfull[s])), "r"(tbytes));
            char* dst = tring + s * tbytes + rank * rows * 128;
            if (C > 1)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                    ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5, %6;" ::"r"(su32(dst)),
                    "l"(&tx), "r"((int)(u % KB) * 64), "r"((int)rank * rows), "r"(su32(&tfull[s])),
                    "h"((uint16_t)((1u << C) - 1)), "l"(keep)
                    : "memory");
            else
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                    " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
                    "l"(&tx), "r"((int)(u % KB) * 64), "r"(0), "r"(su32(&tfull[s])), "l"(keep)
                    : "memory");
        }
    } else if (warp == 2 && lane == 0) {  // "MMA": needs both, releases both
        int acc = 0;
        for (long long u = u0; u < u1; ++u) {
            int i = (int)(u - u0), s = i % stages, ts = i % tstages;
            wait_parity(su32(&full[s]), (i / stages) & 1);
            wait_parity(su32(&tfull[ts]), (i / tstages) & 1);
            acc ^= ((int*)(smem + s * kStage))[0] ^ ((int*)(tring + ts * tbytes))[0];
            asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&empty[s])));
            for (uint32_t r = 0; r < C; ++r)  // this CTA's copy of token stage ts is free
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 mapa(su32(&tempty[ts]), r)));
        }
        if (acc == 0x12345678) *out = acc;
    }
    if (C > 1) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
}

int main() {
    const size_t bytes = 4ull << 30;
    char* p;
    int* out;
    CK(cudaMalloc(&p, bytes));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(p, 1, bytes));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int reps = 1;  // launches back to back between the events
    auto time_it = [&](auto launch) {
        float best = 1e9;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(a);
            for (int i = 0; i < reps; ++i) launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ms /= reps;
            if (ms < best) best = ms;
        }
        return bytes / (best / 1e3) / 1e9;  // bulk variants read (bytes/G rounded down to 32 KB)*G: <0.1% less
    };
    for (int k : {1, 2, 4}) {
        double g = time_it([&] { k_ldg<<<sms * k, 512>>>((const int4*)p, bytes / 16, out); });
        printf("ldg   %d CTA/SM x 512 thr: %.0f GB/s\n", k, g);
    }
    for (int st : {3, 4, 5, 6, 7}) {
        int smem = st * 32768 + 256;
        CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        double g = time_it([&] { k_bulk<<<sms, 160, smem>>>(p, bytes, st, out); });
        printf("bulk  1 CTA/SM, %d x 32 KB stages: %.0f GB/s\n", st, g);
    }
    for (int st : {2, 3}) {
        int smem = st * 32768 + 256;
        double g = time_it([&] { k_bulk<<<sms * 2, 160, smem>>>(p, bytes, st, out); });
        printf("bulk2 2 CTA/SM, %d x 32 KB stages each: %.0f GB/s\n", st, g);
    }
    // 2-D boxes over [rows][K] matrices of the C3 GEMM shapes, 5 stages
    for (int K : {5120, 20480}) {
        const long long rows = (long long)(bytes / 2 / K) / 256 * 256;
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)K * 2};
        cuuint32_t box[2] = {64, 256};
        cuuint32_t estr[2] = {1, 1};
        if (cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
        for (int st : {5, 6}) {
            int smem = st * 32768 + 256 + 1024;
            CK(cudaFuncSetAttribute(k_tma2d, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            double g = time_it([&] { k_tma2d<<<sms, 160, smem>>>(tm, rows / 256, K / 64, st, out); });
            printf("tma2d K=%d box 64x256 SW128, %d stages: %.0f GB/s (of the whole buffer)\n", K, st,
                   g * (double)(rows * K * 2) / bytes);
        }
    }

    // the same weight stream over ONE FC matrix (210 MB), 20 launches back to back
    reps = 20;
    {
        const int K = 5120;
        const long long rows = 20480;
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)K * 2};
        cuuint32_t box[2] = {64, 256}, estr[2] = {1, 1};
        cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        int smem = 5 * 32768 + 256 + 1024;
        CK(cudaFuncSetAttribute(k_tma2d, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        double g = time_it([&] { k_tma2d<<<sms, 160, smem>>>(tm, rows / 256, K / 64, 5, out); });
        printf("tma2d FC matrix 210 MB, 5 stages, x20 back to back: %.0f GB/s\n", g * (double)(rows * K * 2) / bytes);
        double g2 = time_it([&] { k_bulk<<<sms, 160, smem>>>(p, (size_t)rows * K * 2, 5, out); });
        printf("bulk  FC-sized 210 MB, 5 stages, x20 back to back: %.0f GB/s\n", g2 * (double)(rows * K * 2) / bytes);
    }
    // weights + tokens (T x 64 per unit from an L2-resident [T][K] matrix), FC shape
    {
        const int K = 5120;
        const long long rows = 20480;
        CUtensorMap tw, tx;
        cuuint64_t dw[2] = {(cuuint64_t)K, (cuuint64_t)rows}, sw[1] = {(cuuint64_t)K * 2};
        cuuint32_t bw[2] = {64, 256}, es[2] = {1, 1};
        cuTensorMapEncodeTiled(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dw, sw, bw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        char* xp = p + (size_t)rows * K * 2;  // tokens right after the weights
        for (int T : {48, 112, 192}) {
            for (int C : {1, 2, 4}) {
                for (int ts : {2, 4}) {
                    cuuint64_t dx[2] = {(cuuint64_t)K, (cuuint64_t)T}, sx[1] = {(cuuint64_t)K * 2};
                    cuuint32_t bx[2] = {64, (cuuint32_t)(T / C)};
                    cuTensorMapEncodeTiled(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xp, dx, sx, bx, es,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                    int st = (226 * 1024 - 2048 - ts * T * 128) / 32768;
                    if (st > 6) st = 6;
                    int smem = st * 32768 + ts * T * 128 + 2048;
                    CK(cudaFuncSetAttribute(k_wtok, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                    if (C > 1) CK(cudaFuncSetAttribute(k_wtok, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(sms / C * C);
                    cfg.blockDim = dim3(128);
                    cfg.dynamicSmemBytes = smem;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = C;
                    at[0].val.clusterDim.y = 1;
                    at[0].val.clusterDim.z = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = 1;
                    double g = time_it([&] {
                        cudaLaunchKernelEx(&cfg, k_wtok, tw, tx, (long long)(rows / 256), K / 64, T, st, ts, out);
                    });
                    CK(cudaGetLastError());
                    printf("w+tok FC T=%3d cluster %d, %d weight + %d token stages: %.0f GB/s of weights\n", T, C, st,
                           ts, g * (double)(rows * K * 2) / bytes);
                }
            }
        }
    }
    CK(cudaGetLastError());
    return 0;
}
