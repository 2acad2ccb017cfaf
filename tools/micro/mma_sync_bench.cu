// Throughput / latency of legacy mma.sync m16n8k16 bf16 on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int CHAINS>
__global__ void k(float* out, long long* cyc, int iters) {
    float d[CHAINS][4] = {};
    uint32_t a = threadIdx.x * 0x10001u, b = threadIdx.x ^ 0x3f803f80u;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) mma(d[c], a, a + c, a ^ c, a, b, b + c);
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    float* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
    const int iters = 4096;
    for (int warps : {1, 4, 8, 16}) {
        long long h;
        k<1><<<1, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize();
        k<1><<<1, 32 * warps>>>(out, cyc, iters); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("warps/SM %2d chains 1: %.1f cycles per mma per warp (latency-bound)\n", warps, (double)h / iters);
        k<8><<<1, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize();
        k<8><<<1, 32 * warps>>>(out, cyc, iters); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("warps/SM %2d chains 8: %.2f cycles per mma per warp -> SM rate %.2f mma/cycle\n", warps, (double)h / iters / 8, warps * 8.0 * iters / h);
    }
    return 0;
}
