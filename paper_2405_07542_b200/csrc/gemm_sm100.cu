// Weight-streaming tcgen05 GEMM for the packed verify-step token stream.
//
//   Y[t][m] = sum_k W[m][k] * X[t][k]       (W = weights [M][K], X = tokens [T][K])
//
// "Swap-AB": the weights are the 128-row UMMA A operand (M = output features)
// and the T <= 256 packed tokens are the UMMA N dimension, so a CTA tile is
// 256 output features x N tokens held in TMEM as two 128-lane fp32
// accumulators.  Operands are staged by TMA with the 128-byte swizzle into a
// multi-stage mbarrier ring and one thread issues tcgen05.mma.
//
// The GEMM is HBM-bound (every weight byte is read once per step), so the
// schedule is stream-K: the m_tiles x (K/64) k-block units are split evenly
// over the SMs and every CTA streams one contiguous range of weights.  Each
// (tile, contributor) segment dumps its raw fp32 accumulator into a partial
// buffer; a separate, fully parallel reduction kernel sums a tile's
// contributors in fixed order (deterministic) and applies the fused epilogue:
// bias + Q/K/V scatter into the unpadded KV arena, bias + GELU, bias +
// residual + the NEXT LayerNorm, or the LM-head argmax (lowest id on ties).
// No CTA ever waits for another one, and TMEM is double-buffered for N <= 128
// so a segment's epilogue overlaps the next segment's MMAs.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM
// allocator, w4-7 epilogue (TMEM lanes 0-127).
#include <cuda_bf16.h>

#include <string>

#include "../../include/specdec_b200_debug.h"
#include "gemm.h"
#include "sm100_ptx.cuh"

namespace sdb {
namespace {

constexpr int kBM = 256, kBK = 64, kThreads = 256;
constexpr int kABytes = kBM * kBK * 2;  // 32 KB per stage
constexpr int kSmemBytes = 226 * 1024;  // + static smem stays under the 227 KB opt-in limit
constexpr int kMaxStages = 8;

__host__ __device__ __forceinline__ int cta_of(long long x, long long G, long long U) {
    return (int)(((x + 1) * G - 1) / U);
}

__device__ __forceinline__ float gelu_fast(float x) {
    // GELU-tanh (model.cpp:71-74) with the hardware tanh
    const float c = 0.7978845608028654f;
    float u = c * (x + 0.044715f * x * x * x);
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
    return 0.5f * x * (1.0f + t);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB32,
           const __grid_constant__ CUtensorMap tmB64, const __grid_constant__ CUtensorMap tmB128,
           const __grid_constant__ CUtensorMap tmB256, const GemmArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int T = a.dT ? *a.dT : a.T;
    if (T <= 0) return;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int BN = T <= 16 ? 16 : ((T + 15) / 16) * 16;
    const int box = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    const CUtensorMap* tmB = box == 32 ? &tmB32 : box == 64 ? &tmB64 : box == 128 ? &tmB128 : &tmB256;
    const int nbuf = BN <= 128 ? 2 : 1;  // TMEM accumulator buffers
    const int stage_bytes = kABytes + box * 128;
    int S = (kSmemBytes - 2048) / stage_bytes;
    if (S > kMaxStages) S = kMaxStages;
    uint8_t* stage_base = smem;
    uint64_t* bars = (uint64_t*)(smem + S * stage_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kMaxStages;
    uint64_t* tmem_full = bars + 2 * kMaxStages;  // [2]
    uint64_t* tmem_empty = tmem_full + 2;          // [2]
    uint32_t* tmem_slot = (uint32_t*)(tmem_empty + 2);

    const long long KB = a.K / kBK;
    const long long U = (long long)a.m_tiles * KB;
    const long long G = gridDim.x;
    const long long u0 = (long long)blockIdx.x * U / G, u1 = (long long)(blockIdx.x + 1) * U / G;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(tmB);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tmem_full[b], 1);
            ptx::mbar_init(&tmem_empty[b], 128);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer: one contiguous weight range
            const uint64_t pol_w = ptx::policy_evict_first();  // weights: streamed once
            const uint64_t pol_x = ptx::policy_evict_last();   // tokens: re-read by every tile
            int stage = 0;
            uint32_t phase = 0;
            for (long long u = u0; u < u1; ++u) {
                int tile = (int)(u / KB), kb = (int)(u % KB);
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sa = stage_base + stage * stage_bytes;
                ptx::mbar_arrive_expect_tx(&full[stage], stage_bytes);
                ptx::tma_load_2d(sa, &tmA, &full[stage], kb * kBK, tile * kBM, pol_w);
                ptx::tma_load_2d(sa + kABytes, tmB, &full[stage], kb * kBK, 0, pol_x);
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            const uint32_t idesc = ptx::umma_idesc_bf16(128, BN);
            int stage = 0;
            uint32_t phase = 0, seg = 0;
            for (long long u = u0; u < u1; ++seg) {
                int kb0 = (int)(u % KB);
                int kb1 = (int)min((long long)KB, kb0 + (u1 - u));
                const int buf = nbuf == 2 ? (int)(seg & 1) : 0;
                const uint32_t use = nbuf == 2 ? seg >> 1 : seg;
                ptx::mbar_wait(&tmem_empty[buf], (use & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t d0 = tmem + (nbuf == 2 ? buf * 256 : 0);
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    uint32_t sa = ptx::smem_u32(stage_base + stage * stage_bytes);
                    uint32_t sb = sa + kABytes;
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        uint64_t bdesc = ptx::umma_desc_kmajor_sw128(sb + k * 32);
#pragma unroll
                        for (int acc = 0; acc < 2; ++acc) {
                            uint64_t adesc = ptx::umma_desc_kmajor_sw128(sa + acc * (128 * 128) + k * 32);
                            ptx::umma_bf16(d0 + acc * (nbuf == 2 ? 128 : 256), adesc, bdesc, idesc,
                                           (kb > kb0 || k > 0) ? 1u : 0u);
                        }
                    }
                    ptx::umma_commit(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::umma_commit(&tmem_full[buf]);
                u += kb1 - kb0;
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue: TMEM -> fp32 partials
        const int w = warp - 4;
        const int row_in_acc = w * 32 + lane;
        const int ncols = BN;
        uint32_t seg = 0;
        for (long long u = u0; u < u1; ++seg) {
            int tile = (int)(u / KB), kb0 = (int)(u % KB);
            int kb1 = (int)min((long long)KB, kb0 + (u1 - u));
            const int buf = nbuf == 2 ? (int)(seg & 1) : 0;
            const uint32_t use = nbuf == 2 ? seg >> 1 : seg;
            const int ci = (int)blockIdx.x - cta_of((long long)tile * KB, G, U);
            float* dst = a.part + (size_t)(tile * a.max_contrib + ci) * 256 * 256;
            ptx::mbar_wait(&tmem_full[buf], use & 1);
            ptx::tc_fence_after();
            const uint32_t trow = tmem + ((uint32_t)(w * 32) << 16) + (nbuf == 2 ? buf * 256 : 0);
            for (int acc = 0; acc < 2; ++acc) {
                const int row = acc * 128 + row_in_acc;
                for (int j0 = 0; j0 < ncols; j0 += 16) {
                    float v[16];
                    ptx::tmem_ld16(trow + acc * (nbuf == 2 ? 128 : 256) + j0, v);
#pragma unroll
                    for (int i = 0; i < 16; ++i) dst[(size_t)(j0 + i) * 256 + row] = v[i];
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tmem_empty[buf]);
            u += kb1 - kb0;
        }
    }
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------- reductions
struct RedInfo {
    int KB, G;
    long long U;
};

// sum of tile contributors in contributor order (deterministic)
__device__ __forceinline__ float tile_sum(const GemmArgs& a, const RedInfo& r, int tile, int t, int row) {
    long long tk0 = (long long)tile * r.KB;
    int cf = cta_of(tk0, r.G, r.U), cl = cta_of(tk0 + r.KB - 1, r.G, r.U);
    const float* p = a.part + ((size_t)tile * a.max_contrib * 256 + t) * 256 + row;
    float v = 0.0f;
    for (int c = 0; c <= cl - cf; ++c) v += __ldcg(p + (size_t)c * 256 * 256);
    return v;
}

// grid (T_upper, m_tiles), block 256: one output feature per thread
template <int EPI>
__global__ void __launch_bounds__(256) k_reduce_tile(GemmArgs a, RedInfo r) {
    const int t = blockIdx.x, tile = blockIdx.y, row = threadIdx.x;
    const int T = a.dT ? *a.dT : a.T;
    const int m = tile * 256 + row;
    if (t >= T || m >= a.M) return;
    float v = tile_sum(a, r, tile, t, row);
    if constexpr (EPI == EPI_STORE) {
        a.out_f32[(size_t)t * a.ld_out + m] = v;
    } else if constexpr (EPI == EPI_GELU) {
        a.out_bf16[(size_t)t * a.ld_out + m] = __float2bfloat16_rn(gelu_fast(v + a.bias[m]));
    } else if constexpr (EPI == EPI_QKV) {
        __nv_bfloat16 x = __float2bfloat16_rn(v + a.bias[m]);
        int which = m / a.h, hm = m - which * a.h;
        if (which == 0) {
            a.out_bf16[(size_t)t * a.h + hm] = x;
        } else {
            Plan pl = a.plans[t];
            if (pl.store) {
                int head = hm / a.hd, d = hm - head * a.hd;
                size_t off = ((((size_t)a.layer * 2 + (which - 1)) * a.B + pl.sample) * a.heads + head) *
                                 (size_t)a.cap * a.hd +
                             (size_t)pl.write_slot * a.hd + d;
                a.kv[off] = x;
            }
        }
    }
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* scratch) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (threadIdx.x % 32 == 0) scratch[threadIdx.x / 32] = v;
    __syncthreads();
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) s += scratch[i];
    return s;
}

// grid T_upper, block 512: residual add of one token row, then the next
// LayerNorm of that row (two-pass mean / variance, eps 1e-5) -> bf16
constexpr int kLnThreads = 512, kLnPer = 16;  // hidden <= 8192
__global__ void __launch_bounds__(kLnThreads) k_reduce_resid_ln(GemmArgs a, RedInfo r) {
    __shared__ float scratch[32];
    const int t = blockIdx.x;
    const int T = a.dT ? *a.dT : a.T;
    if (t >= T) return;
    float x[kLnPer];
    float s = 0.0f;
    float* res = a.out_f32 + (size_t)t * a.ld_out;
#pragma unroll
    for (int k = 0; k < kLnPer; ++k) {
        int m = threadIdx.x + k * kLnThreads;
        x[k] = 0.0f;
        if (m < a.M) {
            float v = tile_sum(a, r, m >> 8, t, m & 255) + a.bias[m];
            x[k] = res[m] + v;
            res[m] = x[k];
            s += x[k];
        }
    }
    const float mean = block_sum<kLnThreads>(s, scratch) / a.M;
    float q = 0.0f;
#pragma unroll
    for (int k = 0; k < kLnPer; ++k) {
        int m = threadIdx.x + k * kLnThreads;
        if (m < a.M) q += (x[k] - mean) * (x[k] - mean);
    }
    const float inv = rsqrtf(block_sum<kLnThreads>(q, scratch) / a.M + 1e-5f);
    __nv_bfloat16* y = a.ln_out + (size_t)t * a.M;
#pragma unroll
    for (int k = 0; k < kLnPer; ++k) {
        int m = threadIdx.x + k * kLnThreads;
        if (m < a.M) y[m] = __float2bfloat16_rn((x[k] - mean) * inv * a.ln_g[m] + a.ln_b[m]);
    }
}

// grid T_upper, block 1024: greedy_next over the vocab (model.cpp:34-41)
__global__ void __launch_bounds__(1024) k_reduce_argmax(GemmArgs a, RedInfo r) {
    __shared__ float sv[32];
    __shared__ int si[32];
    const int t = blockIdx.x;
    const int T = a.dT ? *a.dT : a.T;
    if (t >= T) return;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    bool bad = false;
    for (int m = threadIdx.x; m < a.vocab; m += 1024) {
        float v = tile_sum(a, r, m >> 8, t, m & 255);
        if (a.logits) a.logits[(size_t)t * a.vocab + m] = v;
        if (!isfinite(v)) bad = true;
        if (v > bv) {  // ascending m per thread: strict > keeps the lowest id
            bv = v;
            bi = m;
        }
    }
    if (bad) atomicExch(a.flag, 1);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    if (threadIdx.x % 32 == 0) {
        sv[threadIdx.x / 32] = bv;
        si[threadIdx.x / 32] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 32; ++w)
            if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) {
                bv = sv[w];
                bi = si[w];
            }
        a.argmax[t] = bi == 0x7fffffff ? 0 : bi;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw Error(INTERNAL, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeFn)p;
    }
    return fn;
}

int max_contrib_for(int m_tiles, int KB, int G) {
    long long U = (long long)m_tiles * KB;
    int mx = 1;
    for (int t = 0; t < m_tiles; ++t) {
        long long tk0 = (long long)t * KB;
        mx = std::max(mx, cta_of(tk0 + KB - 1, G, U) - cta_of(tk0, G, U) + 1);
    }
    return mx;
}

}  // namespace

CUtensorMap make_tmap_2d(const void* base, int64_t rows, int64_t cols, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(INTERNAL, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

void make_b_maps(GemmMaps& maps, const void* x, int64_t rows, int64_t cols) {
    const int boxes[4] = {32, 64, 128, 256};
    for (int i = 0; i < 4; ++i) maps.B[i] = make_tmap_2d(x, rows, cols, boxes[i]);
}

void gemm_plan(GemmArgs& a, int sms) {
    SD_CHECK(a.K % kBK == 0, CONFIG, "bf16 mode needs K % 64 == 0");
    long long U = (long long)a.m_tiles * (a.K / kBK);
    a.grid = (int)std::min<long long>(U, sms);
    a.max_contrib = max_contrib_for(a.m_tiles, a.K / kBK, a.grid);
}

size_t gemm_part_floats(int M, int K, int sms) {
    GemmArgs a{};
    a.M = M;
    a.K = K;
    a.m_tiles = (M + 255) / 256;
    gemm_plan(a, sms);
    return (size_t)a.m_tiles * a.max_contrib * 256 * 256;
}

void gemm_prepare() {
    CUDA_OK(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
}

void gemm_launch(int epi, const GemmArgs& a, const GemmMaps& maps, int T_upper, cudaStream_t st) {
    static bool prepared = false;
    if (!prepared) {
        gemm_prepare();
        prepared = true;
    }
    SD_CHECK(T_upper <= 256, INTERNAL, "GEMM token tile is at most 256");
    k_gemm<<<a.grid, kThreads, kSmemBytes, st>>>(maps.A, maps.B[0], maps.B[1], maps.B[2], maps.B[3], a);
    RedInfo r{a.K / kBK, a.grid, (long long)a.m_tiles * (a.K / kBK)};
    switch (epi) {
        case EPI_STORE: k_reduce_tile<EPI_STORE><<<dim3(T_upper, a.m_tiles), 256, 0, st>>>(a, r); break;
        case EPI_GELU: k_reduce_tile<EPI_GELU><<<dim3(T_upper, a.m_tiles), 256, 0, st>>>(a, r); break;
        case EPI_QKV: k_reduce_tile<EPI_QKV><<<dim3(T_upper, a.m_tiles), 256, 0, st>>>(a, r); break;
        case EPI_RESID_LN: k_reduce_resid_ln<<<T_upper, kLnThreads, 0, st>>>(a, r); break;
        case EPI_ARGMAX: k_reduce_argmax<<<T_upper, 1024, 0, st>>>(a, r); break;
        default: throw Error(INTERNAL, "unknown GEMM epilogue");
    }
    CUDA_OK(cudaGetLastError());
}

}  // namespace sdb

// --------------------------------------------------------------- test hook
namespace {
thread_local std::string g_dbg_err;
}
extern "C" int sd_debug_gemm(const uint16_t* W, const uint16_t* X, int M, int K, int T, int grid, float* Y,
                             float* usec) {
    using namespace sdb;
    try {
        int m_tiles = (M + 255) / 256;
        size_t wbytes = (size_t)m_tiles * 256 * K * 2, xbytes = (size_t)T * K * 2;
        void *dW = dmalloc(wbytes), *dX = dmalloc(xbytes), *dY = dmalloc((size_t)T * M * 4);
        GemmArgs a{};
        a.M = M;
        a.K = K;
        a.m_tiles = m_tiles;
        a.T = T;
        gemm_plan(a, grid > 0 ? grid : 148);
        void* dpart = dmalloc(sizeof(float) * (size_t)m_tiles * a.max_contrib * 256 * 256);
        CUDA_OK(cudaMemset(dW, 0, wbytes));
        CUDA_OK(cudaMemcpy(dW, W, (size_t)M * K * 2, cudaMemcpyHostToDevice));
        CUDA_OK(cudaMemcpy(dX, X, xbytes, cudaMemcpyHostToDevice));
        GemmMaps maps;
        maps.A = make_tmap_2d(dW, (int64_t)m_tiles * 256, K, 256);
        make_b_maps(maps, dX, T, K);
        a.part = (float*)dpart;
        a.out_f32 = (float*)dY;
        a.ld_out = M;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        gemm_launch(EPI_STORE, a, maps, T, 0);  // warm-up / configure
        CUDA_OK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        gemm_launch(EPI_STORE, a, maps, T, 0);
        cudaEventRecord(e1);
        CUDA_OK(cudaDeviceSynchronize());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (usec) *usec = ms * 1000.0f;
        CUDA_OK(cudaMemcpy(Y, dY, (size_t)T * M * 4, cudaMemcpyDeviceToHost));
        dfree(dW);
        dfree(dX);
        dfree(dY);
        dfree(dpart);
        return 0;
    } catch (const Error& e) {
        g_dbg_err = e.what();
        return e.code;
    }
}
