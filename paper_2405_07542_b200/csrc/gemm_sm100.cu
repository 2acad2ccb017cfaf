// Weight-streaming tcgen05 GEMM for the packed verify-step token stream.
//
//   Y[t][m] = sum_k W[m][k] * X[t][k]       (W = weights [M][K], X = tokens [T][K])
//
// "Swap-AB": the weights are the 128-row UMMA A operand (M = output features)
// and the T <= 256 packed tokens are the UMMA N dimension, so one CTA tile is
// 256 output features x N tokens held in TMEM as two 128-lane fp32
// accumulators (512 columns).  Operands are staged by TMA with the 128-byte
// swizzle into a multi-stage mbarrier ring; one thread issues tcgen05.mma.
//
// The problem is HBM-bound (every weight byte is read once per step), so the
// schedule is stream-K: the m_tiles x n_tiles x (K/64) k-block units are split
// evenly over the 148 SMs; a tile cut by a CTA boundary is reduced by its last
// finishing contributor, in contributor order (deterministic), which then runs
// the fused epilogue: bias, GELU, residual add, Q/K/V scatter into the
// unpadded KV arena, or the LM-head (max, lowest id) argmax partials.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM
// allocator, w4-7 epilogue (TMEM lanes 0-127).
#include <cuda_bf16.h>

#include "gemm.h"
#include "sm100_ptx.cuh"

namespace sdb {
namespace {

constexpr int kBM = 256, kBK = 64, kThreads = 256;
constexpr int kABytes = kBM * kBK * 2;  // 32 KB per stage
constexpr int kRedBytes = 8 * 256 * 8;  // argmax cross-warp scratch
constexpr int kSmemBytes = 226 * 1024;  // + static smem stays under the 227 KB opt-in limit
constexpr int kMaxStages = 8;

struct Seg {
    int tile, kb0, kb1;
};

__device__ __forceinline__ int cta_of(long long x, long long G, long long U) {
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

template <int EPI>
__device__ __forceinline__ void finalize_chunk(const GemmArgs& a, int T, int m_base, int n0, int j0, int acc,
                                               int lane, int w, float (&v)[16], float* red_val, int* red_idx) {
    const int m = m_base + acc * 128 + w * 32 + lane;
    if constexpr (EPI == EPI_STORE) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            int j = n0 + j0 + i;
            if (j < T && m < a.M) a.out_f32[(size_t)j * a.ld_out + m] = v[i];
        }
    } else if constexpr (EPI == EPI_RESID) {
        float b = (m < a.M && a.bias) ? a.bias[m] : 0.0f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            int j = n0 + j0 + i;
            if (j < T && m < a.M) a.out_f32[(size_t)j * a.ld_out + m] += v[i] + b;
        }
    } else if constexpr (EPI == EPI_GELU) {
        float b = (m < a.M && a.bias) ? a.bias[m] : 0.0f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            int j = n0 + j0 + i;
            if (j < T && m < a.M) a.out_bf16[(size_t)j * a.ld_out + m] = __float2bfloat16_rn(gelu_fast(v[i] + b));
        }
    } else if constexpr (EPI == EPI_QKV) {
        if (m < a.M) {
            float b = a.bias ? a.bias[m] : 0.0f;
            int which = m / a.h, hm = m - which * a.h;
            int head = hm / a.hd, d = hm - head * a.hd;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                int j = n0 + j0 + i;
                if (j >= T) break;
                __nv_bfloat16 x = __float2bfloat16_rn(v[i] + b);
                if (which == 0) {
                    a.out_bf16[(size_t)j * a.h + hm] = x;
                } else {
                    Plan pl = a.plans[j];
                    if (pl.store) {
                        size_t off = ((((size_t)a.layer * 2 + (which - 1)) * a.B + pl.sample) * a.heads + head) *
                                         (size_t)a.cap * a.hd +
                                     (size_t)pl.write_slot * a.hd + d;
                        a.kv[off] = x;
                    }
                }
            }
        }
    } else if constexpr (EPI == EPI_ARGMAX) {
        const bool valid = m < a.vocab;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            int j = n0 + j0 + i;
            float x = v[i];
            if (valid && j < T) {
                if (a.logits) a.logits[(size_t)j * a.vocab + m] = x;
                if (!isfinite(x)) atomicExch(a.flag, 1);
            }
            float bv = valid ? x : -INFINITY;
            int bi = valid ? m : 0x7fffffff;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            if (lane == 0) {
                red_val[(w * 2 + acc) * 256 + j0 + i] = bv;
                red_idx[(w * 2 + acc) * 256 + j0 + i] = bi;
            }
        }
    }
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB32,
           const __grid_constant__ CUtensorMap tmB64, const __grid_constant__ CUtensorMap tmB128,
           const __grid_constant__ CUtensorMap tmB256, const GemmArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int T = a.dT ? *a.dT : a.T;
    if (T <= 0) return;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int n_tiles = (T + 255) / 256;
    int BN = n_tiles > 1 ? 256 : ((T + 15) / 16) * 16;
    const int box = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    if (n_tiles == 1 && BN < 16) BN = 16;
    const CUtensorMap* tmB = box == 32 ? &tmB32 : box == 64 ? &tmB64 : box == 128 ? &tmB128 : &tmB256;
    const int stage_bytes = kABytes + box * 128;
    const int avail = kSmemBytes - 1024 - kRedBytes - 1024;
    int S = avail / stage_bytes;
    if (S > kMaxStages) S = kMaxStages;
    uint8_t* stage_base = smem;
    float* red_val = (float*)(smem + S * stage_bytes);
    int* red_idx = (int*)((uint8_t*)red_val + 8 * 256 * 4);  // [8][256] floats, then [8][256] ints
    uint64_t* bars = (uint64_t*)((uint8_t*)red_val + kRedBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kMaxStages;
    uint64_t* tmem_full = bars + 2 * kMaxStages;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = (uint32_t*)(tmem_empty + 1);
    __shared__ int s_last;

    const long long KB = a.K / kBK;
    const long long U = (long long)a.m_tiles * n_tiles * KB;
    const long long G = gridDim.x;
    const long long u0 = (long long)blockIdx.x * U / G, u1 = (long long)(blockIdx.x + 1) * U / G;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(tmB);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(tmem_full, 1);
        ptx::mbar_init(tmem_empty, 128);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            const uint64_t pol_w = ptx::policy_evict_first();  // weights: streamed once
            const uint64_t pol_x = ptx::policy_evict_last();   // tokens: re-read by every tile
            int stage = 0;
            uint32_t phase = 0;
            for (long long u = u0; u < u1;) {
                int tile = (int)(u / KB), kb0 = (int)(u % KB);
                int kb1 = (int)min((long long)KB, kb0 + (u1 - u));
                int m0 = (tile % a.m_tiles) * kBM, n0 = (tile / a.m_tiles) * 256;
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = stage_base + stage * stage_bytes;
                    ptx::mbar_arrive_expect_tx(&full[stage], stage_bytes);
                    ptx::tma_load_2d(sa, &tmA, &full[stage], kb * kBK, m0, pol_w);
                    ptx::tma_load_2d(sa + kABytes, tmB, &full[stage], kb * kBK, n0, pol_x);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                u += kb1 - kb0;
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
                ptx::mbar_wait(tmem_empty, (seg & 1) ^ 1);
                ptx::tc_fence_after();
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
                            ptx::umma_bf16(tmem + acc * 256, adesc, bdesc, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                        }
                    }
                    ptx::umma_commit(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::umma_commit(tmem_full);
                u += kb1 - kb0;
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue
        const int w = warp - 4;
        const int et = threadIdx.x - 128;  // 0..127
        uint32_t seg = 0;
        for (long long u = u0; u < u1; ++seg) {
            int tile = (int)(u / KB), kb0 = (int)(u % KB);
            int kb1 = (int)min((long long)KB, kb0 + (u1 - u));
            int m_tile = tile % a.m_tiles, n_tile = tile / a.m_tiles;
            int m_base = m_tile * kBM, n0 = n_tile * 256;
            int ncols = min(BN, ((T - n0 + 15) / 16) * 16);
            bool whole = kb0 == 0 && kb1 == KB;
            ptx::mbar_wait(tmem_full, seg & 1);
            ptx::tc_fence_after();
            const uint32_t trow = tmem + ((uint32_t)(w * 32) << 16);
            if (whole) {
                for (int acc = 0; acc < 2; ++acc)
                    for (int j0 = 0; j0 < ncols; j0 += 16) {
                        float v[16];
                        ptx::tmem_ld16(trow + acc * 256 + j0, v);
                        finalize_chunk<EPI>(a, T, m_base, n0, j0, acc, lane, w, v, red_val, red_idx);
                    }
                ptx::tc_fence_before();
                ptx::mbar_arrive(tmem_empty);
            } else {
                // split tile: publish this contributor's partial, the last one reduces
                long long tk0 = (long long)tile * KB;
                int cf = cta_of(tk0, G, U), cl = cta_of(tk0 + KB - 1, G, U);
                int me = blockIdx.x;
                int slot = me == cf ? 2 * me + 1 : 2 * me;
                float* mine = a.ws + (size_t)slot * 256 * 256;
                for (int acc = 0; acc < 2; ++acc)
                    for (int j0 = 0; j0 < ncols; j0 += 16) {
                        float v[16];
                        ptx::tmem_ld16(trow + acc * 256 + j0, v);
#pragma unroll
                        for (int i = 0; i < 16; ++i) mine[(size_t)(j0 + i) * 256 + acc * 128 + et] = v[i];
                    }
                ptx::tc_fence_before();
                ptx::mbar_arrive(tmem_empty);
                __threadfence();
                ptx::named_bar_sync(1, 128);
                if (et == 0) {
                    int old = atomicAdd(&a.counters[tile], 1);
                    s_last = (old == cl - cf);
                    if (s_last) atomicExch(&a.counters[tile], 0);
                }
                ptx::named_bar_sync(1, 128);
                if (s_last) {
                    __threadfence();
                    for (int acc = 0; acc < 2; ++acc)
                        for (int j0 = 0; j0 < ncols; j0 += 16) {
                            float v[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i) v[i] = 0.0f;
                            for (int c = cf; c <= cl; ++c) {
                                const float* p = a.ws + (size_t)(c == cf ? 2 * c + 1 : 2 * c) * 256 * 256;
#pragma unroll
                                for (int i = 0; i < 16; ++i) v[i] += __ldcg(p + (size_t)(j0 + i) * 256 + acc * 128 + et);
                            }
                            finalize_chunk<EPI>(a, T, m_base, n0, j0, acc, lane, w, v, red_val, red_idx);
                        }
                }
            }
            if constexpr (EPI == EPI_ARGMAX) {
                ptx::named_bar_sync(1, 128);
                bool fin = whole || s_last;
                if (fin) {
                    for (int j = et; j < ncols; j += 128) {
                        float bv = red_val[j];
                        int bi = red_idx[j];
                        for (int g = 1; g < 8; ++g) {
                            float ov = red_val[g * 256 + j];
                            int oi = red_idx[g * 256 + j];
                            if (ov > bv || (ov == bv && oi < bi)) {
                                bv = ov;
                                bi = oi;
                            }
                        }
                        if (n0 + j < T) {
                            a.part_val[(size_t)m_tile * a.ld_part + n0 + j] = bv;
                            a.part_idx[(size_t)m_tile * a.ld_part + n0 + j] = bi;
                        }
                    }
                }
                ptx::named_bar_sync(1, 128);
            }
            u += kb1 - kb0;
        }
    }
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc<512>(tmem);
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

template <int EPI>
void launch_impl(const GemmArgs& a, const GemmMaps& maps, int grid, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        CUDA_OK(cudaFuncSetAttribute(k_gemm<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
        configured = true;
    }
    k_gemm<EPI><<<grid, kThreads, kSmemBytes, st>>>(maps.A, maps.B[0], maps.B[1], maps.B[2], maps.B[3], a);
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

void gemm_prepare() {
    CUDA_OK(cudaFuncSetAttribute(k_gemm<EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    CUDA_OK(cudaFuncSetAttribute(k_gemm<EPI_RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    CUDA_OK(cudaFuncSetAttribute(k_gemm<EPI_GELU>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    CUDA_OK(cudaFuncSetAttribute(k_gemm<EPI_QKV>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    CUDA_OK(cudaFuncSetAttribute(k_gemm<EPI_ARGMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
}

int gemm_grid(const GemmArgs& a, int T_upper, int sms) {
    long long n_tiles = (T_upper + 255) / 256;
    long long U = (long long)a.m_tiles * n_tiles * (a.K / kBK);
    return (int)(U < sms ? U : sms);
}

void gemm_launch(int epi, const GemmArgs& a, const GemmMaps& maps, int grid, cudaStream_t st) {
    SD_CHECK(a.K % kBK == 0, CONFIG, "bf16 mode needs K % 64 == 0");
    switch (epi) {
        case EPI_STORE: launch_impl<EPI_STORE>(a, maps, grid, st); break;
        case EPI_RESID: launch_impl<EPI_RESID>(a, maps, grid, st); break;
        case EPI_GELU: launch_impl<EPI_GELU>(a, maps, grid, st); break;
        case EPI_QKV: launch_impl<EPI_QKV>(a, maps, grid, st); break;
        case EPI_ARGMAX: launch_impl<EPI_ARGMAX>(a, maps, grid, st); break;
        default: throw Error(INTERNAL, "unknown GEMM epilogue");
    }
    CUDA_OK(cudaGetLastError());
}

}  // namespace sdb

// --------------------------------------------------------------- test hook
#include "../../include/specdec_b200_debug.h"
#include <string>
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
        void* dws = dmalloc((size_t)2 * 148 * 256 * 256 * 4);
        int* dcnt = (int*)dmalloc(65536 * 4);
        CUDA_OK(cudaMemset(dW, 0, wbytes));
        CUDA_OK(cudaMemset(dcnt, 0, 65536 * 4));
        CUDA_OK(cudaMemcpy(dW, W, (size_t)M * K * 2, cudaMemcpyHostToDevice));
        CUDA_OK(cudaMemcpy(dX, X, xbytes, cudaMemcpyHostToDevice));
        GemmMaps maps;
        maps.A = make_tmap_2d(dW, (int64_t)m_tiles * 256, K, 256);
        make_b_maps(maps, dX, T, K);
        GemmArgs a{};
        a.M = M;
        a.K = K;
        a.m_tiles = m_tiles;
        a.T = T;
        a.ws = (float*)dws;
        a.counters = dcnt;
        a.out_f32 = (float*)dY;
        a.ld_out = M;
        int g = grid > 0 ? grid : gemm_grid(a, T, 148);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        gemm_launch(EPI_STORE, a, maps, g, 0);  // warm-up / configure
        CUDA_OK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        gemm_launch(EPI_STORE, a, maps, g, 0);
        cudaEventRecord(e1);
        CUDA_OK(cudaDeviceSynchronize());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (usec) *usec = ms * 1000.0f;
        CUDA_OK(cudaMemcpy(Y, dY, (size_t)T * M * 4, cudaMemcpyDeviceToHost));
        dfree(dW); dfree(dX); dfree(dY); dfree(dws); dfree(dcnt);
        return 0;
    } catch (const Error& e) {
        g_dbg_err = e.what();
        return e.code;
    }
}
