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

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/specdec_b200_debug.h"
#include "gemm.h"
#include "pdl.cuh"
#include "sm100_ptx.cuh"
#include "trace.cuh"

SD_TRACE_TU(gemm)

#ifdef SD_GEMM_PROBE  // bottleneck probes (tools/gemm_probe.py --probe): never in the library build
#define PROBE(bit) ((a.probe & (bit)) != 0)
#else
#define PROBE(bit) false
#endif

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

// Partial-sum buffer layout: [tile * max_contrib + contributor][256 tokens][256 rows] fp32.
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB32,
           const __grid_constant__ CUtensorMap tmB64, const __grid_constant__ CUtensorMap tmB128,
           const __grid_constant__ CUtensorMap tmB256, const GemmArgs a) {
    CtaTrace trace__(TK_GEMM);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // smem layout from the host-side token bound (known before the predecessor
    // finishes); the true token count is read after griddepcontrol.wait
    const int box = a.box;                 // host bound: sizes the token-ring stages
    // Decoupled rings: the weight (A) ring is as deep as smem allows so enough
    // HBM bytes stay in flight to cover DRAM latency; the token (B) ring is
    // shallow because B is L2-resident (re-read by every tile).
    const int b_bytes = box * 128;         // stage stride (the loaded box may be smaller)
    const int SB = 2;
    int SA = (kSmemBytes - 2048 - SB * b_bytes) / kABytes;
    if (SA > kMaxStages) SA = kMaxStages;
    uint8_t* a_base = smem;
    uint8_t* b_base = smem + SA * kABytes;
    uint64_t* bars = (uint64_t*)(b_base + SB * b_bytes);
    uint64_t* fullA = bars;
    uint64_t* emptyA = bars + kMaxStages;
    uint64_t* fullB = bars + 2 * kMaxStages;       // [SB]
    uint64_t* emptyB = fullB + 4;                  // [SB]
    uint64_t* tmem_full = emptyB + 4;              // [2]
    uint64_t* tmem_empty = tmem_full + 2;          // [2]
    uint32_t* tmem_slot = (uint32_t*)(tmem_empty + 2);

    const long long KB = a.K / kBK;
    const long long U = (long long)a.m_tiles * KB;
    const long long G = gridDim.x;
    const long long u0 = (long long)blockIdx.x * U / G, u1 = (long long)(blockIdx.x + 1) * U / G;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        for (int s = 0; s < SA; ++s) {
            ptx::mbar_init(&fullA[s], 1);
            ptx::mbar_init(&emptyA[s], 1);
        }
        for (int s = 0; s < SB; ++s) {
            ptx::mbar_init(&fullB[s], 1);
            ptx::mbar_init(&emptyB[s], 1);
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
    pdl_trigger();

    if (warp == 0) {
        // ---------------- TMA producer A: one contiguous weight range.  Weights
        // do not depend on earlier kernels, so this starts BEFORE
        // griddepcontrol.wait and the ring fills while the predecessor drains.
        if (lane == 0) {
            const uint64_t pol_w = ptx::policy_evict_first();  // weights: streamed once
            int stage = 0;
            uint32_t phase = 0;
            for (long long u = u0; u < u1; ++u) {
                ptx::mbar_wait(&emptyA[stage], phase ^ 1);
                uint8_t* sa = a_base + stage * kABytes;
                ptx::mbar_arrive_expect_tx(&fullA[stage], kABytes);
                ptx::tma_load_2d(sa, &tmA, &fullA[stage], (int)(u % KB) * kBK, (int)(u / KB) * kBM, pol_w);
                if (++stage == SA) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else {
        pdl_wait();  // tokens, partial buffer and token count come from earlier kernels
        const int T = a.dT ? *a.dT : a.T;
        const int BN = T <= 16 ? 16 : ((T + 15) / 16) * 16;
        const bool idle = T <= 0 || BN > box;  // a finished step: drain the A ring only
        // the token box and TMEM double-buffering follow the TRUE token count:
        // a device-resident step sized for B x (k+1) tokens usually carries far fewer
        const int box_d = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
        const CUtensorMap* tmB = box_d == 32 ? &tmB32 : box_d == 64 ? &tmB64 : box_d == 128 ? &tmB128 : &tmB256;
        const int nbuf = box_d <= 128 ? 2 : 1;  // TMEM accumulator buffers
        if (warp == 3) {
            if (lane == 0 && !idle && !PROBE(2)) {  // ---------------- TMA producer B: the token tile of each k-block
                const uint64_t pol_x = ptx::policy_evict_last();  // tokens: re-read by every tile
                int stage = 0;
                uint32_t phase = 0;
                for (long long u = u0; u < u1; ++u) {
                    ptx::mbar_wait(&emptyB[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&fullB[stage], box_d * 128);
                    ptx::tma_load_2d(b_base + stage * b_bytes, tmB, &fullB[stage], (int)(u % KB) * kBK, 0, pol_x);
                    if (++stage == SB) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        } else if (warp == 1) {
            if (lane == 0) {  // ---------------- MMA issuer
                const uint32_t idesc = ptx::umma_idesc_bf16(128, BN);
                int sa_i = 0, sb_i = 0;
                uint32_t pa = 0, pb = 0, seg = 0;
                for (long long u = u0; u < u1; ++seg) {
                    int kb0 = (int)(u % KB);
                    int kb1 = (int)min((long long)KB, kb0 + (u1 - u));
                    const int buf = nbuf == 2 ? (int)(seg & 1) : 0;
                    const uint32_t use = nbuf == 2 ? seg >> 1 : seg;
                    if (!idle) {
                        ptx::mbar_wait(&tmem_empty[buf], (use & 1) ^ 1);
                        ptx::tc_fence_after();
                    }
                    const uint32_t d0 = tmem + (nbuf == 2 ? buf * 256 : 0);
                    for (int kb = kb0; kb < kb1; ++kb) {
                        ptx::mbar_wait(&fullA[sa_i], pa);
                        if (!idle) {
                            if (!PROBE(2)) ptx::mbar_wait(&fullB[sb_i], pb);
                            ptx::tc_fence_after();
                            uint32_t sa = ptx::smem_u32(a_base + sa_i * kABytes);
                            uint32_t sb = ptx::smem_u32(b_base + sb_i * b_bytes);
#pragma unroll
                            for (int k = 0; k < (PROBE(1) ? 0 : kBK / 16); ++k) {
                                uint64_t bdesc = ptx::umma_desc_kmajor_sw128(sb + k * 32);
#pragma unroll
                                for (int acc = 0; acc < 2; ++acc) {
                                    uint64_t adesc = ptx::umma_desc_kmajor_sw128(sa + acc * (128 * 128) + k * 32);
                                    ptx::umma_bf16(d0 + acc * (nbuf == 2 ? 128 : 256), adesc, bdesc, idesc,
                                                   (kb > kb0 || k > 0) ? 1u : 0u);
                                }
                            }
                            ptx::umma_commit(&emptyB[sb_i]);
                            if (++sb_i == SB) {
                                sb_i = 0;
                                pb ^= 1;
                            }
                        }
                        ptx::umma_commit(&emptyA[sa_i]);
                        if (++sa_i == SA) {
                            sa_i = 0;
                            pa ^= 1;
                        }
                    }
                    if (!idle) ptx::umma_commit(&tmem_full[buf]);
                    u += kb1 - kb0;
                }
            }
        } else if (warp >= 4 && !idle) {  // ---------------- epilogue: TMEM -> fp32 partials
            const int w = warp - 4;
            const int row_in_acc = w * 32 + lane;
            const uint64_t pol_keep = ptx::policy_evict_last();  // partials are re-read from L2
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
                    float* dcol = dst + acc * 128 + row_in_acc;  // [token][row]: a warp stores 128 B per token
                    for (int j0 = 0; j0 < BN; j0 += 16) {
                        float v[16];
                        ptx::tmem_ld16(trow + acc * (nbuf == 2 ? 128 : 256) + j0, v);
                        if (!PROBE(4)) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                ptx::st_f32_hint(dcol + (size_t)(j0 + i) * 256, v[i], pol_keep);
                        }
                    }
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&tmem_empty[buf]);
                u += kb1 - kb0;
            }
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

__device__ __forceinline__ void tile_contrib(const RedInfo& r, int tile, int& n) {
    long long tk0 = (long long)tile * r.KB;
    n = cta_of(tk0 + r.KB - 1, r.G, r.U) - cta_of(tk0, r.G, r.U) + 1;
}

// grid (m_tiles, ceil(T_upper / RT)), block 256: thread = one output feature
// (tile row) for RT consecutive tokens, read as float4; contributors summed in
// order (deterministic).
// tokens per reduction thread: 8 (2 for the residual GEMMs, whose ~8
// contributors per tile make every token a long sum) -- same-box A/B:
// (16, 4) 8.29 ms -> (8, 2) 8.19 ms per C3 step
constexpr int kRT = 8;
template <int EPI, int RT = kRT>
__global__ void __launch_bounds__(256) k_reduce_tile(const GemmArgs a, const RedInfo r) {
    CtaTrace trace__(EPI == EPI_STORE ? TK_RED_STORE : EPI == EPI_GELU ? TK_RED_GELU : EPI == EPI_QKV ? TK_RED_QKV : TK_RED_RESID);
    pdl_trigger();
    pdl_wait();
    const int tile = blockIdx.x, t0 = blockIdx.y * RT, row = threadIdx.x;
    const int T = a.dT ? *a.dT : a.T;
    const int m = tile * 256 + row;
    if (t0 >= T || m >= a.M) return;
    int nc;
    tile_contrib(r, tile, nc);
    const float* __restrict__ p = a.part + ((size_t)tile * a.max_contrib * 256 + t0) * 256 + row;
    const int nt = min(RT, T - t0);
    // independent of the partials: issued before them, so the residual
    // read-modify-write and the bias cost no extra L2 round trip
    const float b = a.bias ? a.bias[m] : 0.0f;
    float old[RT];
    if constexpr (EPI == EPI_RESID_LN) {
#pragma unroll
        for (int i = 0; i < RT; ++i) old[i] = i < nt ? a.out_f32[(size_t)(t0 + i) * a.ld_out + m] : 0.0f;
    }
    float v[RT];
#pragma unroll
    for (int i = 0; i < RT; ++i) v[i] = 0.0f;
    // every load of CB contributors x RT tokens is issued before the first add:
    // one L2 round trip per CB contributors instead of one per contributor
    // (the sum itself still runs in contributor order: deterministic)
    constexpr int CB = RT <= 4 ? 8 : 4;
    for (int c0 = 0; c0 < nc; c0 += CB) {
        float x[CB][RT];
#pragma unroll
        for (int cc = 0; cc < CB; ++cc)
#pragma unroll
            for (int i = 0; i < RT; ++i)
                x[cc][i] = (c0 + cc < nc && i < nt) ? __ldcg(p + ((size_t)(c0 + cc) * 256 + i) * 256) : 0.0f;
#pragma unroll
        for (int cc = 0; cc < CB; ++cc)
#pragma unroll
            for (int i = 0; i < RT; ++i)
                if (c0 + cc < nc) v[i] += x[cc][i];
    }
    if constexpr (EPI == EPI_RESID_LN) {  // residual add; the LayerNorm runs in k_ln_rows
#pragma unroll
        for (int i = 0; i < RT; ++i)
            if (i < nt) a.out_f32[(size_t)(t0 + i) * a.ld_out + m] = old[i] + (v[i] + b);
    } else if constexpr (EPI == EPI_QKV) {
        const int which = m / a.h, hm = m - which * a.h;
        const int head = hm / a.hd, d = hm - head * a.hd;
#pragma unroll
        for (int i = 0; i < RT; ++i) {
            if (i >= nt) break;
            const int t = t0 + i;
            __nv_bfloat16 x = __float2bfloat16_rn(v[i] + b);
            if (which == 0) {
                a.out_bf16[(size_t)t * a.h + hm] = x;
            } else {
                Plan pl = a.plans[t];
                if (pl.store) {
                    size_t off = ((((size_t)a.layer * 2 + (which - 1)) * a.B + pl.sample) * a.heads + head) *
                                     (size_t)a.cap * a.hd +
                                 (size_t)pl.write_slot * a.hd + d;
                    a.kv[off] = x;
                }
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < RT; ++i) {
            if (i >= nt) break;
            const int t = t0 + i;
            if constexpr (EPI == EPI_STORE) a.out_f32[(size_t)t * a.ld_out + m] = v[i];
            if constexpr (EPI == EPI_GELU)
                a.out_bf16[(size_t)t * a.ld_out + m] = __float2bfloat16_rn(gelu_fast(v[i] + b));
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

// grid T_upper, block 256: LayerNorm of the updated residual row -> bf16
// (two-pass mean / variance, eps 1e-5; hidden <= 8192)
__global__ void __launch_bounds__(256) k_ln_rows(const GemmArgs a) {
    CtaTrace trace__(TK_LN_ROWS);
    pdl_trigger();
    pdl_wait();
    __shared__ float scratch[32];
    const int t = blockIdx.x;
    const int T = a.dT ? *a.dT : a.T;
    if (t >= T) return;
    const float4* __restrict__ row = (const float4*)(a.out_f32 + (size_t)t * a.ld_out);
    constexpr int kPer = 8;  // float4 per thread
    float4 x[kPer], g[kPer], bb[kPer];
    float s = 0.0f;
    const int n4 = a.M / 4;
    const float4* g4 = (const float4*)a.ln_g;
    const float4* b4 = (const float4*)a.ln_b;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {  // gamma / beta in flight with the row: one L2 round trip
        const int i = threadIdx.x + k * 256;
        x[k] = i < n4 ? row[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        g[k] = i < n4 ? g4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        bb[k] = i < n4 ? b4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) s += x[k].x + x[k].y + x[k].z + x[k].w;
    const float mean = block_sum<256>(s, scratch) / a.M;
    float q = 0.0f;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = threadIdx.x + k * 256;
        if (i < n4) {
            float dx = x[k].x - mean, dy = x[k].y - mean, dz = x[k].z - mean, dw = x[k].w - mean;
            q += dx * dx + dy * dy + dz * dz + dw * dw;
        }
    }
    const float inv = rsqrtf(block_sum<256>(q, scratch) / a.M + 1e-5f);
    __nv_bfloat162* y = (__nv_bfloat162*)(a.ln_out + (size_t)t * a.M);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = threadIdx.x + k * 256;
        if (i < n4) {
            y[2 * i] = __floats2bfloat162_rn((x[k].x - mean) * inv * g[k].x + bb[k].x,
                                             (x[k].y - mean) * inv * g[k].y + bb[k].y);
            y[2 * i + 1] = __floats2bfloat162_rn((x[k].z - mean) * inv * g[k].z + bb[k].z,
                                                 (x[k].w - mean) * inv * g[k].w + bb[k].w);
        }
    }
}

// grid (ceil(T_upper / 4), ceil(m_tiles / kArgTiles)), block 256: LM-head
// logits of 4 tokens over kArgTiles vocab tiles, reduced to (max, lowest id)
// partials per token; the last block of a token (arrival counter) folds them
// into greedy_next (model.cpp:34-41).
constexpr int kArgTiles = 8;
__global__ void __launch_bounds__(256) k_reduce_argmax(const GemmArgs a, const RedInfo r, float* __restrict__ pv,
                                                       int* __restrict__ pi, int* __restrict__ cnt) {
    CtaTrace trace__(TK_ARGMAX);
    pdl_trigger();
    pdl_wait();
    __shared__ float sv[8][4];
    __shared__ int si[8][4];
    __shared__ int s_last[4];
    const int t0 = blockIdx.x * 4, grp = blockIdx.y, row = threadIdx.x;
    const int T = a.dT ? *a.dT : a.T;
    if (t0 >= T) return;
    const int nt = min(4, T - t0);
    float bv[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int bi[4] = {0x7fffffff, 0x7fffffff, 0x7fffffff, 0x7fffffff};
    bool bad = false;
    // Partials of kTB tiles x <= kCB contributors x 4 tokens are loaded before the
    // first add (one L2 round trip per kTB tiles instead of one per tile and
    // contributor); each tile still sums its contributors in order from 0
    constexpr int kTB = 4, kCB = 4;
    for (int k0 = 0; k0 < kArgTiles; k0 += kTB) {
        float x[kTB][kCB][4];
        int ncs[kTB];
#pragma unroll
        for (int kk = 0; kk < kTB; ++kk) {
            const int tile = grp * kArgTiles + k0 + kk;
            ncs[kk] = 0;
            if (tile < a.m_tiles) tile_contrib(r, tile, ncs[kk]);
            const float* p = a.part + ((size_t)tile * a.max_contrib * 256 + t0) * 256 + row;
#pragma unroll
            for (int c = 0; c < kCB; ++c)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    x[kk][c][i] = (c < ncs[kk] && i < nt) ? __ldcg(p + (size_t)c * 65536 + i * 256) : 0.0f;
        }
#pragma unroll
        for (int kk = 0; kk < kTB; ++kk) {  // ascending ids per thread: strict > keeps the lowest
            const int tile = grp * kArgTiles + k0 + kk;
            const int m = tile * 256 + row;
            if (tile >= a.m_tiles) break;
            float vv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int c = 0; c < kCB; ++c)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (c < ncs[kk]) vv[i] += x[kk][c][i];
            if (ncs[kk] > kCB) {  // more contributors than one batch (not at C2-C5 shapes)
                const float* p = a.part + ((size_t)tile * a.max_contrib * 256 + t0) * 256 + row;
                for (int c = kCB; c < ncs[kk]; ++c)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (i < nt) vv[i] += __ldcg(p + (size_t)c * 65536 + i * 256);
            }
            if (m >= a.vocab) continue;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (i >= nt) break;
                if (a.logits) a.logits[(size_t)(t0 + i) * a.vocab + m] = vv[i];
                if (!isfinite(vv[i])) bad = true;
                if (vv[i] > bv[i]) {
                    bv[i] = vv[i];
                    bi[i] = m;
                }
            }
        }
    }
    if (bad) atomicExch(a.flag, 1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            float ov = __shfl_xor_sync(0xffffffffu, bv[i], off);
            int oi = __shfl_xor_sync(0xffffffffu, bi[i], off);
            if (ov > bv[i] || (ov == bv[i] && oi < bi[i])) {
                bv[i] = ov;
                bi[i] = oi;
            }
        }
        if (threadIdx.x % 32 == 0) {
            sv[threadIdx.x / 32][i] = bv[i];
            si[threadIdx.x / 32][i] = bi[i];
        }
    }
    __syncthreads();
    if (threadIdx.x < nt) {
        const int i = threadIdx.x, t = t0 + i;
        float b = sv[0][i];
        int idx = si[0][i];
        for (int w = 1; w < 8; ++w)
            if (sv[w][i] > b || (sv[w][i] == b && si[w][i] < idx)) {
                b = sv[w][i];
                idx = si[w][i];
            }
        pv[(size_t)t * gridDim.y + grp] = b;
        pi[(size_t)t * gridDim.y + grp] = idx;
        __threadfence();
        const int old = atomicAdd(&cnt[t], 1);
        s_last[i] = old == (int)gridDim.y - 1;
    }
    __syncthreads();
    if (threadIdx.x < nt && s_last[threadIdx.x]) {
        const int t = t0 + threadIdx.x;
        __threadfence();
        float best = __ldcg(pv + (size_t)t * gridDim.y);
        int bidx = __ldcg(pi + (size_t)t * gridDim.y);
        for (int k = 1; k < (int)gridDim.y; ++k) {
            float ov = __ldcg(pv + (size_t)t * gridDim.y + k);
            int oi = __ldcg(pi + (size_t)t * gridDim.y + k);
            if (ov > best || (ov == best && oi < bidx)) {
                best = ov;
                bidx = oi;
            }
        }
        a.argmax[t] = bidx == 0x7fffffff ? 0 : bidx;
        cnt[t] = 0;  // self-resetting for the next launch / graph replay
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
    // at least kMinUnits k-blocks (128 KB of weights) per CTA: a small GEMM
    // (e.g. a 125M-parameter draft model) otherwise splits every tile over a
    // dozen CTAs and pays more in partials and reduction than in streaming
    constexpr long long kMinUnits = 4;
    a.grid = (int)std::max<long long>(1, std::min<long long>((U + kMinUnits - 1) / kMinUnits, sms));
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
    if (first_use_on_device(2))
        CUDA_OK(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
}

void gemm_launch(int epi, const GemmArgs& a, const GemmMaps& maps, int T_upper, cudaStream_t st,
                 cudaEvent_t after_stream) {
    gemm_prepare();
    SD_CHECK(T_upper <= 256, INTERNAL, "GEMM token tile is at most 256");
    GemmArgs ab = a;
    ab.box = T_upper <= 32 ? 32 : T_upper <= 64 ? 64 : T_upper <= 128 ? 128 : 256;
    launch_k(k_gemm, dim3(a.grid), dim3(kThreads), kSmemBytes, st, maps.A, maps.B[0], maps.B[1], maps.B[2],
             maps.B[3], ab);
    if (after_stream) CUDA_OK(cudaEventRecord(after_stream, st));
    RedInfo r{a.K / kBK, a.grid, (long long)a.m_tiles * (a.K / kBK)};
    const dim3 tg(a.m_tiles, (T_upper + kRT - 1) / kRT);
    switch (epi) {
        case EPI_STORE: launch_k(k_reduce_tile<EPI_STORE>, tg, dim3(256), 0, st, ab, r); break;
        case EPI_GELU: launch_k(k_reduce_tile<EPI_GELU>, tg, dim3(256), 0, st, ab, r); break;
        case EPI_QKV: launch_k(k_reduce_tile<EPI_QKV>, tg, dim3(256), 0, st, ab, r); break;
        case EPI_RESID_LN:  // tile-parallel split-K sum + residual, then the row LayerNorm
            SD_CHECK(a.M % 4 == 0 && a.M <= 8192, CONFIG, "bf16 mode needs hidden % 4 == 0 and <= 8192");
            launch_k(k_reduce_tile<EPI_RESID_LN, 2>, dim3(a.m_tiles, (T_upper + 1) / 2), dim3(256), 0, st, ab, r);
            launch_k(k_ln_rows, dim3(T_upper), dim3(256), 0, st, ab);
            break;
        case EPI_ARGMAX: {
            const int groups = (a.m_tiles + kArgTiles - 1) / kArgTiles;
            SD_CHECK(groups <= kArgmaxGroups, CONFIG, "vocab too large for the argmax scratch");
            SD_CHECK(a.am.val && a.am.idx && a.am.cnt, INTERNAL, "argmax scratch missing");
            launch_k(k_reduce_argmax, dim3((T_upper + 3) / 4, groups), dim3(256), 0, st, ab, r, a.am.val, a.am.idx,
                     a.am.cnt);
            break;
        }
        case -1: break;  // probe: streaming kernel only
        default: throw Error(INTERNAL, "unknown GEMM epilogue");
    }
    CUDA_OK(cudaGetLastError());
}

void ln_rows_launch(const GemmArgs& a, int T_upper, cudaStream_t st) {
    SD_CHECK(a.M % 4 == 0 && a.M <= 8192, CONFIG, "bf16 mode needs hidden % 4 == 0 and <= 8192");
    launch_k(k_ln_rows, dim3(T_upper), dim3(256), 0, st, a);
}

}  // namespace sdb

// --------------------------------------------------------------- test hook
namespace {
thread_local std::string g_dbg_err;
}
extern "C" int sd_debug_gemm(const uint16_t* W, const uint16_t* X, int M, int K, int T, int grid, int flags,
                             float* Y, float* usec) {
    // flags bit3: time the streaming kernel alone (no reduction; Y is not written)
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
        gemm_plan(a, grid > 0 ? grid : device_sm_count());
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
        const int epi = (flags & 8) ? -1 : EPI_STORE;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        a.probe = flags >> 4;  // only a -DSD_GEMM_PROBE build reads it
        gemm_launch(epi, a, maps, T, 0);  // warm-up / configure
        CUDA_OK(cudaDeviceSynchronize());
        const int reps = (flags & 128) ? 10 : 1;  // bit 7: ten launches back to back, mean
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) gemm_launch(epi, a, maps, T, 0);
        cudaEventRecord(e1);
        CUDA_OK(cudaDeviceSynchronize());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (usec) *usec = ms * 1000.0f;
        if (epi == EPI_STORE) CUDA_OK(cudaMemcpy(Y, dY, (size_t)T * M * 4, cudaMemcpyDeviceToHost));
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

// --------------------------------------------------------------- timeline hook
namespace sdb {
void trace_set_fast(const TraceBuf& b);
void trace_set_step(const TraceBuf& b);
void trace_set_gemmcl(const TraceBuf& b);
}  // namespace sdb
namespace {
sdb::TraceBuf g_host_trace{nullptr, nullptr, 0};
void trace_set_all(const sdb::TraceBuf& b) {
    sdb::trace_set_gemm(b);
    sdb::trace_set_fast(b);
    sdb::trace_set_step(b);
    sdb::trace_set_gemmcl(b);
}
}  // namespace
extern "C" int sd_debug_trace_begin(int cap) {
    using namespace sdb;
    try {
        if (g_host_trace.rec) {
            dfree(g_host_trace.rec);
            dfree(g_host_trace.count);
        }
        g_host_trace.rec = (TraceRec*)dmalloc(sizeof(TraceRec) * (size_t)cap);
        g_host_trace.count = (unsigned*)dmalloc(sizeof(unsigned));
        g_host_trace.cap = (unsigned)cap;
        CUDA_OK(cudaMemset(g_host_trace.count, 0, sizeof(unsigned)));
        trace_set_all(g_host_trace);
        CUDA_OK(cudaDeviceSynchronize());
        return 0;
    } catch (const Error& e) {
        g_dbg_err = e.what();
        return e.code;
    }
}
extern "C" int sd_debug_trace_end(void* out, int cap, int* n) {
    using namespace sdb;
    try {
        CUDA_OK(cudaDeviceSynchronize());
        unsigned cnt = 0;
        if (g_host_trace.count) CUDA_OK(cudaMemcpy(&cnt, g_host_trace.count, sizeof(cnt), cudaMemcpyDeviceToHost));
        cnt = std::min<unsigned>(cnt, std::min<unsigned>((unsigned)cap, g_host_trace.cap));
        if (cnt) CUDA_OK(cudaMemcpy(out, g_host_trace.rec, sizeof(TraceRec) * cnt, cudaMemcpyDeviceToHost));
        *n = (int)cnt;
        trace_set_all(TraceBuf{nullptr, nullptr, 0});
        return 0;
    } catch (const Error& e) {
        g_dbg_err = e.what();
        return e.code;
    }
}
