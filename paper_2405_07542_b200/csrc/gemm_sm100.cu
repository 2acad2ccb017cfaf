// Weight-streaming tcgen05 GEMM for the packed verify-step token stream.
//
//   Y[t][m] = sum_k W[m][k] * X[t][k]       (W = weights [M][K], X = tokens [T][K])
//
// "Swap-AB": the weights are the 128-row UMMA A operand (M = output features)
// and the T <= 256 packed tokens are the UMMA N dimension, so a CTA tile is
// 128 output features x N tokens held in TMEM as one fp32 accumulator,
// double-buffered (2 x 256 columns) so a segment's epilogue overlaps the next
// segment's MMAs.  Operands are staged by TMA with the 128-byte swizzle into
// mbarrier rings -- a deep weight (A) ring, because every weight byte comes
// from HBM exactly once per step, and a shallow token (B) ring, because the
// token tile is L2-resident -- and one thread issues tcgen05.mma.
//
// The GEMM is HBM-bound, so the schedule is stream-K: the m_tiles x (K/64)
// k-block units are split evenly over one CTA per SM and every CTA streams a
// contiguous range of weights.  Each (tile, contributor) segment dumps its raw
// fp32 accumulator into an L2-resident partial buffer and bumps the tile's
// arrival counter; the epilogue warps of every CTA then reduce an equal share
// of the GEMM's (tile, token) outputs (waiting for each tile's contributors),
// summing contributors in a fixed order (deterministic), and apply the fused
// epilogue: bias + Q/K/V scatter into the unpadded KV arena, bias + GELU,
// bias + residual and -- after a grid-wide arrival count -- the NEXT
// LayerNorm, or the LM-head (max, lowest id) argmax.  No reduction or
// LayerNorm kernels exist.
//
// Persistent chains: one launch streams up to four dependent GEMMs (O-proj ->
// FC -> PROJ -> next layer's QKV, or ... -> LM head).  The weight producer
// never waits on data, so GEMM i+1's weights stream into the ring while GEMM i
// is still being reduced and normalised; only its token-operand loads wait
// for a grid-wide "GEMM i done" count.  HBM therefore stays busy across the
// GEMM boundaries that used to cost a kernel drain + ramp each.
//
// Co-residency of the waits: the grid is <= one CTA per SM and every CTA
// triggers its dependents only after it is resident, so every CTA a wait
// depends on is running or done; each role processes the chain in order and
// only ever waits on strictly earlier work (partials are published before a
// CTA's own reductions, reductions before the done count), so there is no
// cycle.
//
// Warp roles (384 threads): w0 TMA producer (weights), w1 MMA issuer, w2 TMEM
// allocator, w3 TMA producer (tokens), w4-11 epilogue: TMEM drain (two warps
// per 32-lane TMEM quadrant, alternate 16-column chunks), reduction jobs,
// LayerNorm rows, argmax folds.
#include <cuda_bf16.h>

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

namespace sdb {
namespace {

constexpr int kBM = kGemmTile, kBK = 64, kThreads = 384, kEpiThreads = 256;
constexpr int kABytes = kBM * kBK * 2;    // 16 KB per weight stage
constexpr int kSmemBytes = 225 * 1024;    // + ~1.1 KB static smem stays under the 227 KB opt-in limit
constexpr int kMaxStagesA = 16, kMaxStagesB = 8;
constexpr size_t kSlot = 256 * kBM;       // floats per (tile, contributor) partial: [256 tok][128 rows]
constexpr int kLnCnt = kGemmMaxTiles;     // counter index: finished reduction slices (LN barrier)
constexpr int kDoneCnt = kGemmMaxTiles + 1; // counter index: CTAs done with the GEMM (chain dependency)
constexpr int kTokCnt = 768;              // counter index base: per-token argmax arrivals [256]

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

// Counter polls are RELAXED loads (an ld.acquire.gpu compiles to a load plus
// an L1 invalidate, which -- issued thousands of times by a spinning thread --
// stalls the SM's memory pipe for the warps doing real work); one acquire
// fence after the count is reached orders the subsequent reads.
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_count(const int* p, int target, int sleep_ns = 64) {
    while (ld_relaxed(p) < target) __nanosleep(sleep_ns);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

struct Seg {
    int tile, kb0, kb1, ci, nc;
};
// the k-block range of a CTA that starts at unit u, and its tile's contributors
__device__ __forceinline__ Seg seg_at(long long u, long long u1, long long KB, long long G, long long U) {
    Seg s;
    s.tile = (int)(u / KB);
    s.kb0 = (int)(u % KB);
    s.kb1 = (int)min(KB, (long long)s.kb0 + (u1 - u));
    if (U < G) {  // every CTA owns at most one unit: one contributor per k-block
        s.ci = s.kb0;
        s.nc = (int)KB;
        return s;
    }
    const long long tk0 = (long long)s.tile * KB;
    const int c0 = cta_of(tk0, G, U);
    s.ci = (int)blockIdx.x - c0;
    s.nc = cta_of(tk0 + KB - 1, G, U) - c0 + 1;
    return s;
}

// sum over the 256 epilogue threads (warps 4-11, named barrier 1)
__device__ __forceinline__ float epi_sum(float v, float* scratch) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    ptx::named_bar_sync(1, kEpiThreads);
    if (threadIdx.x % 32 == 0) scratch[threadIdx.x / 32 - 4] = v;
    ptx::named_bar_sync(1, kEpiThreads);
    float t = 0.0f;
#pragma unroll
    for (int w = 0; w < kEpiThreads / 32; ++w) t += scratch[w];
    return t;
}

// LayerNorm of one updated fp32 residual row -> bf16 (two-pass mean /
// variance, eps 1e-5, model.cpp:57-69; hidden <= 8192, % 4 == 0) by the
// 256 epilogue threads
__device__ __forceinline__ void ln_row(const GemmArgs& a, int t, float* scratch) {
    const int tid = threadIdx.x - 128;
    const float4* __restrict__ row = (const float4*)(a.out_f32 + (size_t)t * a.ld_out);
    constexpr int kPer = 8;  // float4 per thread
    float4 x[kPer];
    float s = 0.0f;
    const int n4 = a.M / 4;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = tid + k * kEpiThreads;
        x[k] = i < n4 ? __ldcg(row + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        s += x[k].x + x[k].y + x[k].z + x[k].w;
    }
    const float mean = epi_sum(s, scratch) / a.M;
    float q = 0.0f;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = tid + k * kEpiThreads;
        if (i < n4) {
            float dx = x[k].x - mean, dy = x[k].y - mean, dz = x[k].z - mean, dw = x[k].w - mean;
            q += dx * dx + dy * dy + dz * dz + dw * dw;
        }
    }
    const float inv = rsqrtf(epi_sum(q, scratch + 8) / a.M + 1e-5f);
    __nv_bfloat162* y = (__nv_bfloat162*)(a.ln_out + (size_t)t * a.M);
    const float4* g4 = (const float4*)a.ln_g;
    const float4* b4 = (const float4*)a.ln_b;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = tid + k * kEpiThreads;
        if (i < n4) {
            float4 g = __ldg(g4 + i), b = __ldg(b4 + i);
            y[2 * i] = __floats2bfloat162_rn((x[k].x - mean) * inv * g.x + b.x, (x[k].y - mean) * inv * g.y + b.y);
            y[2 * i + 1] =
                __floats2bfloat162_rn((x[k].z - mean) * inv * g.z + b.z, (x[k].w - mean) * inv * g.w + b.w);
        }
    }
}

__device__ __forceinline__ bool arg_better(float v, int i, float bv, int bi) {
    return v > bv || (v == bv && i < bi);
}

struct Range {
    long long KB, U, u0, u1;
};
__device__ __forceinline__ Range range_of(const GemmArgs& g, long long G) {
    Range r;
    r.KB = g.K / kBK;
    r.U = (long long)g.m_tiles * r.KB;
    r.u0 = (long long)blockIdx.x * r.U / G;
    r.u1 = (long long)(blockIdx.x + 1) * r.U / G;
    return r;
}

// Reduction work is balanced over ALL CTAs, not over a tile's contributors:
// the (tile, token) outputs of a GEMM, tile-major, are split into G equal
// contiguous ranges and a CTA reduces its range in jobs -- tokens [t0, t0+nt)
// of one tile, summed over that tile's nc contributors -- of what one staging
// buffer holds.  `first`: the job starts a new tile (wait for its
// contributors); `staged`: the contributor chunks fit a staging buffer.
struct RJob {
    int tile, nc, t0, nt, first, staged;
};
__device__ __forceinline__ int tile_contributors(int tile, long long KB, long long G, long long U) {
    if (U < G) return (int)KB;  // every CTA owns at most one unit
    const long long tk0 = (long long)tile * KB;
    return cta_of(tk0 + KB - 1, G, U) - cta_of(tk0, G, U) + 1;
}
__device__ __forceinline__ bool rjob_next(const Range& r, long long& x, long long x_end, int& prev_tile, RJob& j,
                                          long long G, int T, uint32_t stg_half, int extra, int dbg) {
    if (x >= x_end) {
        j.nt = 0;
        return false;
    }
    const int tile = (int)(x / T), tok = (int)(x - (long long)tile * T);
    const int nc = tile_contributors(tile, r.KB, G, r.U);
    const int cap = (int)(stg_half / (uint32_t)((nc + extra) * kBM * 4));
    j.tile = tile;
    j.nc = nc;
    j.t0 = tok;
    j.staged = cap >= 1 && !(dbg & 4);
    j.nt = (int)min((long long)min(j.staged ? cap : 8, T - tok), x_end - x);
    j.first = tile != prev_tile;
    prev_tile = tile;
    x += j.nt;
    return true;
}

struct ChainParams {
    CUtensorMap A[kMaxChain];  // weights, box {64, 128}
    CUtensorMap B[kMaxChain];  // token operand, box {64, box}
    int n, T, box, sb, dbg, prefetch;
    const int* dT;
    GemmArgs g[kMaxChain];
};

// Partial-sum buffer layout: [tile * max_contrib + contributor][256 tokens][128 rows] fp32.
__global__ void __launch_bounds__(kThreads, 1) k_gemm(const __grid_constant__ ChainParams P) {
    CtaTrace trace__(TK_GEMM);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ float s_red[16];
    __shared__ int s_last[256];
    __shared__ int s_nlast;
    __shared__ RJob s_job[2];
    __shared__ volatile int s_a_prog;  // weight units the A producer has issued (L2 prefetcher pacing)
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // smem layout from the host-side token bound (known before the predecessor
    // finishes); the true token count is read after griddepcontrol.wait
    const int box = P.box;
    const int b_bytes = box * 128;
    // token stages are >= 16 KB apart: the B ring doubles as the reduction's
    // staging area (two halves) while a GEMM is reduced
    const int b_stride = max(b_bytes, 16384);
    const int SB = P.sb > 0 ? min(P.sb, kMaxStagesB) : 3;
    const uint32_t stg_half = (uint32_t)(SB * b_stride / 2) & ~15u;
    bool has_arg = false;
    for (int i = 0; i < P.n; ++i) has_arg |= P.g[i].epi == EPI_ARGMAX;
    const int scratch_bytes = has_arg ? 2 * 16 * kBM * 4 : 0;  // argmax: [half][16 tokens][128 rows] fp32
    int SA = (kSmemBytes - 2048 - SB * b_stride - scratch_bytes) / kABytes;
    if (SA > kMaxStagesA) SA = kMaxStagesA;
    uint8_t* a_base = smem;
    uint8_t* b_base = smem + SA * kABytes;
    float* arg_scratch = (float*)(b_base + SB * b_stride);
    uint64_t* bars = (uint64_t*)(b_base + SB * b_stride + scratch_bytes);
    uint64_t* fullA = bars;
    uint64_t* emptyA = fullA + kMaxStagesA;
    uint64_t* fullB = emptyA + kMaxStagesA;
    uint64_t* emptyB = fullB + kMaxStagesB;
    uint64_t* tmem_full = emptyB + kMaxStagesB;  // [2]
    uint64_t* tmem_empty = tmem_full + 2;        // [2]
    uint64_t* red_full = tmem_empty + 2;         // [2] staging buffers
    uint32_t* tmem_slot = (uint32_t*)(red_full + 2);
    const long long G = gridDim.x;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < P.n; ++i) {
            ptx::prefetch_tmap(&P.A[i]);
            ptx::prefetch_tmap(&P.B[i]);
        }
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
            ptx::mbar_init(&tmem_empty[b], kEpiThreads);
            ptx::mbar_init(&red_full[b], 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
    if (threadIdx.x == 0) s_a_prog = 0;
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_trigger();

    if (warp == 0) {
        // ---------------- TMA producer A: every GEMM's contiguous weight range,
        // back to back.  Weights never depend on earlier work, so this starts
        // BEFORE griddepcontrol.wait and runs ahead across GEMM boundaries,
        // bounded only by the ring.
        if (lane == 0) {
            const uint64_t pol_w = ptx::policy_evict_first();  // weights: streamed once
            int stage = 0;
            uint32_t phase = 0;
            for (int gi = 0; gi < P.n; ++gi) {
                const Range r = range_of(P.g[gi], G);
                trace_point(101, blockIdx.x | (gi << 16));
                for (long long u = r.u0; u < r.u1; ++u) {
                    ptx::mbar_wait(&emptyA[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&fullA[stage], kABytes);
                    ptx::tma_load_2d(a_base + stage * kABytes, &P.A[gi], &fullA[stage], (int)(u % r.KB) * kBK,
                                     (int)(u / r.KB) * kBM, pol_w);
                    s_a_prog = s_a_prog + 1;
                    if (++stage == SA) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        __syncwarp();
        pdl_wait();
    } else if (warp == 2) {
        // ---------------- L2 prefetcher: keeps HBM streaming when the smem ring
        // is full because the MMA waits at a GEMM boundary (reduction,
        // LayerNorm, dependency count): weight tiles up to kPrefetch units
        // beyond the ring are pulled into L2, so the A loads that follow the
        // boundary hit L2 and the ring refills at L2 speed.
        if (lane == 0 && P.prefetch > 0) {
            int idx = 0;
            for (int gi = 0; gi < P.n; ++gi) {
                const Range r = range_of(P.g[gi], G);
                for (long long u = r.u0; u < r.u1; ++u, ++idx) {
                    if (idx < SA) continue;  // the ring's first fill needs no prefetch
                    while (idx >= s_a_prog + P.prefetch) __nanosleep(128);
                    ptx::tma_prefetch_l2_2d(&P.A[gi], (int)(u % r.KB) * kBK, (int)(u / r.KB) * kBM);
                }
            }
        }
        __syncwarp();
        pdl_wait();
    } else {
        pdl_wait();  // tokens, counters and the token count come from earlier kernels
        const int T = P.dT ? *P.dT : P.T;
        const int BN = T <= 16 ? 16 : ((T + 15) / 16) * 16;
        const bool idle = T <= 0 || BN > box;  // a finished step: drain the A ring only
        if (warp == 3) {
            if (lane == 0 && !idle) {  // ---------------- TMA producer B: the token tile of each k-block
                const uint64_t pol_x = ptx::policy_evict_last();  // tokens: re-read by every tile
                int stage = 0;
                uint32_t phase = 0;
                for (int gi = 0; gi < P.n; ++gi) {
                    const Range r = range_of(P.g[gi], G);
                    if (gi > 0 && r.u0 < r.u1) {
                        // the token operand of GEMM gi is the output of GEMM gi-1
                        wait_count(P.g[gi - 1].cnt + kDoneCnt, (int)G, 32);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    trace_point(102, blockIdx.x | (gi << 16));
                    for (long long u = r.u0; u < r.u1; ++u) {
                        ptx::mbar_wait(&emptyB[stage], phase ^ 1);
                        ptx::mbar_arrive_expect_tx(&fullB[stage], b_bytes);
                        ptx::tma_load_2d(b_base + stage * b_stride, &P.B[gi], &fullB[stage], (int)(u % r.KB) * kBK, 0,
                                         pol_x);
                        if (++stage == SB) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        } else if (warp == 1) {
            if (lane == 0) {  // ---------------- MMA issuer
                const uint32_t idesc = ptx::umma_idesc_bf16(kBM, BN);
                int sa_i = 0, sb_i = 0;
                uint32_t pa = 0, pb = 0, seg = 0;
                for (int gi = 0; gi < P.n; ++gi) {
                    const Range r = range_of(P.g[gi], G);
                    for (long long u = r.u0; u < r.u1; ++seg) {
                        const int kb0 = (int)(u % r.KB);
                        const int kb1 = (int)min(r.KB, kb0 + (r.u1 - u));
                        const int buf = (int)(seg & 1);
                        if (!idle) {
                            ptx::mbar_wait(&tmem_empty[buf], ((seg >> 1) & 1) ^ 1);
                            ptx::tc_fence_after();
                        }
                        const uint32_t d0 = tmem + buf * 256;
                        for (int kb = kb0; kb < kb1; ++kb) {
                            ptx::mbar_wait(&fullA[sa_i], pa);
                            if (!idle) {
                                ptx::mbar_wait(&fullB[sb_i], pb);
                                ptx::tc_fence_after();
                                const uint32_t sa = ptx::smem_u32(a_base + sa_i * kABytes);
                                const uint32_t sb = ptx::smem_u32(b_base + sb_i * b_stride);
                                if (!(P.dbg & 1)) {
#pragma unroll
                                    for (int k = 0; k < kBK / 16; ++k)
                                        ptx::umma_bf16(d0, ptx::umma_desc_kmajor_sw128(sa + k * 32),
                                                       ptx::umma_desc_kmajor_sw128(sb + k * 32), idesc,
                                                       (kb > kb0 || k > 0) ? 1u : 0u);
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
                    trace_point(103, blockIdx.x | (gi << 16));
                }
            }
        } else if (warp >= 4 && !idle) {
            // ---------------- epilogue warps (4-11): TMEM lane quadrant warp % 4 =
            // tile rows, column half (warp - 4) / 4 = alternate 16-token chunks.
            // Per segment:
            //   * not the tile's owner (it does not hold k-block 0): drain the
            //     accumulator into the partial buffer and publish it;
            //   * owner, sole contributor: the epilogue straight from TMEM;
            //   * owner of a split tile -- always its CTA's LAST segment, and in
            //     stream-K order every other contributor but the middle ones has
            //     published long before -- add the others' partials (bulk-copied
            //     into the then idle token ring, two token chunks in flight) to
            //     the accumulator and apply the epilogue.
            // The owner's own accumulator never leaves the SM.
            const int q4 = warp % 4, half = (warp - 4) / 4;
            const int row = q4 * 32 + lane, etid = threadIdx.x - 128;
            const uint64_t pol_keep = ptx::policy_evict_last();    // partials are re-read from L2
            const uint64_t pol_part = ptx::policy_evict_first();   // ... once
            uint32_t seg = 0;
            uint32_t red_ph[2] = {0u, 0u};  // staging-buffer mbarrier phases
            float* scr = arg_scratch + half * 16 * kBM;            // argmax: this half's [16 tok][128 rows]
            for (int gi = 0; gi < P.n; ++gi) {
                const GemmArgs& a = P.g[gi];
                const Range r = range_of(a, G);
                const int extra = a.epi == EPI_RESID_LN ? 1 : 0;    // residual rows staged after the partials
                if (a.epi == EPI_ARGMAX && etid == 0) s_nlast = 0;
                ptx::named_bar_sync(1, kEpiThreads);
                for (long long u = r.u0; u < r.u1; ++seg) {
                    const Seg s = seg_at(u, r.u1, r.KB, G, r.U);
                    u += s.kb1 - s.kb0;
                    const int buf = (int)(seg & 1);
                    ptx::mbar_wait(&tmem_full[buf], (seg >> 1) & 1);
                    ptx::tc_fence_after();
                    const uint32_t trow = tmem + ((uint32_t)(q4 * 32) << 16) + buf * 256;
                    const bool owner = a.owner_mode && s.ci == 0 && a.epi >= 0;
                    if (!owner) {
                        // ---- contributor: accumulator -> partial slot, publish
                        float* dst = a.part + (size_t)(s.tile * a.max_contrib + s.ci) * kSlot + row;  // [token][row]
                        for (int j0 = half * 16; j0 < BN; j0 += 32) {
                            float v[16];
                            ptx::tmem_ld16(trow + j0, v);
                            if (!(P.dbg & 2)) {
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    ptx::st_f32_hint(dst + (size_t)(j0 + i) * kBM, v[i], pol_keep);
                            }
                        }
                        ptx::tc_fence_before();
                        ptx::mbar_arrive(&tmem_empty[buf]);
                        if (a.epi >= 0) {
                            ptx::named_bar_sync(1, kEpiThreads);
                            if (etid == 0) {
                                __threadfence();
                                atomicAdd(a.cnt + s.tile, 1);
                            }
                            __syncwarp();
                        }
                        continue;
                    }
                    // ---- owner: per-row epilogue constants
                    const int m = s.tile * kBM + row;
                    const bool mv = m < a.M;
                    const float bias = (a.bias && mv) ? __ldg(a.bias + m) : 0.0f;
                    int which = 0, hm = m;
                    size_t kv_base = 0, kv_sample = 0;
                    if (a.epi == EPI_QKV && mv) {
                        which = m / a.h;
                        hm = m - which * a.h;
                        const int head = hm / a.hd, d = hm - head * a.hd;
                        kv_sample = (size_t)a.heads * a.cap * a.hd;
                        kv_base = ((size_t)a.layer * 2 + (which > 0 ? which - 1 : 0)) * a.B * kv_sample +
                                  (size_t)head * a.cap * a.hd + d;
                    }
                    // one 16-token chunk [t0, t0+16) of this row: v = accumulator (+ others),
                    // rres = staged residual row values (or null: read from global)
                    auto out16 = [&](int t0, float (&v)[16], const float* rres) {
                        if (a.epi == EPI_ARGMAX) {
                            // rows -> per-token (max, lowest id) through this half's scratch
#pragma unroll
                            for (int i = 0; i < 16; ++i) scr[i * kBM + row] = v[i] + bias;
                            ptx::named_bar_sync(2 + half, 128);
                            const int ht = (etid & 127) / 8, hq = (etid & 127) % 8;  // 8 threads per token
                            const int t = t0 + ht;
                            float bv = -INFINITY;
                            int bi = 0x7fffffff;
                            bool bad = false;
                            if (t < T) {
                                for (int k = 0; k < 16; ++k) {
                                    const int rr = hq * 16 + ((k + ht) & 15);
                                    const int mm = s.tile * kBM + rr;
                                    const float x = scr[ht * kBM + rr];
                                    if (mm < a.vocab) {
                                        if (a.logits) a.logits[(size_t)t * a.vocab + mm] = x;
                                        if (!isfinite(x)) bad = true;
                                        if (arg_better(x, mm, bv, bi)) {
                                            bv = x;
                                            bi = mm;
                                        }
                                    }
                                }
                            }
#pragma unroll
                            for (int off = 1; off < 8; off <<= 1) {
                                const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                                const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                                if (arg_better(ov, oi, bv, bi)) {
                                    bv = ov;
                                    bi = oi;
                                }
                            }
                            if (bad) atomicExch(a.flag, 1);
                            if (hq == 0 && t < T) {
                                a.arg_v[(size_t)t * kGemmMaxTiles + s.tile] = bv;
                                a.arg_i[(size_t)t * kGemmMaxTiles + s.tile] = bi;
                                __threadfence();
                                if (atomicAdd(a.cnt + kTokCnt + t, 1) == a.m_tiles - 1) s_last[atomicAdd(&s_nlast, 1)] = t;
                            }
                            ptx::named_bar_sync(2 + half, 128);  // scratch reuse
                            return;
                        }
                        if (!mv) return;
                        if (a.epi == EPI_RESID_LN) {
                            float rv[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (t0 + i < T)
                                    rv[i] = rres ? rres[i * kBM] : __ldcg(a.out_f32 + (size_t)(t0 + i) * a.ld_out + m);
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (t0 + i < T) a.out_f32[(size_t)(t0 + i) * a.ld_out + m] = rv[i] + v[i] + bias;
                        } else if (a.epi == EPI_GELU) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (t0 + i < T)
                                    a.out_bf16[(size_t)(t0 + i) * a.ld_out + m] = __float2bfloat16_rn(gelu_fast(v[i] + bias));
                        } else if (a.epi == EPI_QKV) {
                            if (which == 0) {
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    if (t0 + i < T) a.out_bf16[(size_t)(t0 + i) * a.h + hm] = __float2bfloat16_rn(v[i] + bias);
                            } else {
                                int slot[16];
#pragma unroll
                                for (int i = 0; i < 16; ++i) {
                                    slot[i] = -1;
                                    if (t0 + i < T) {
                                        const Plan pl = a.plans[t0 + i];
                                        slot[i] = pl.store ? pl.sample * a.cap + pl.write_slot : -1;
                                    }
                                }
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    if (slot[i] >= 0) {
                                        const int smp = slot[i] / a.cap, ws = slot[i] - smp * a.cap;
                                        a.kv[kv_base + (size_t)smp * kv_sample + (size_t)ws * a.hd] =
                                            __float2bfloat16_rn(v[i] + bias);
                                    }
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (t0 + i < T) a.out_f32[(size_t)(t0 + i) * a.ld_out + m] = v[i] + bias;
                        }
                    };
                    if (s.nc == 1) {
                        // ---- sole contributor: epilogue straight from TMEM
                        for (int j0 = half * 16; j0 < BN; j0 += 32) {
                            float v[16];
                            ptx::tmem_ld16(trow + j0, v);
                            out16(j0, v, nullptr);
                        }
                        if (a.epi == EPI_ARGMAX && (BN / 16) % 2 == 1 && half == 1) {
                            // keep the two halves' argmax barriers paired: half 1 has one chunk fewer
                            float v[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i) v[i] = -INFINITY;
                            out16(BN, v, nullptr);
                        }
                    } else {
                        // ---- owner of a split tile: others' partials (slots 1..nc-1) staged per
                        // token chunk into the idle token ring, two chunks in flight
                        const int nothers = s.nc - 1;
                        int cap = (int)(stg_half / (uint32_t)((nothers + extra) * kBM * 4)) & ~15;
                        const bool staged = cap >= 16 && !(P.dbg & 4);
                        if (!staged) cap = 32;
                        const int njobs = (T + cap - 1) / cap;
                        auto issue = [&](int jn) {  // etid 0: job jn into staging buffer jn & 1
                            const int b2 = jn & 1;
                            if (jn >= njobs) return;
                            if (jn == 0) {
                                trace_point(109, blockIdx.x | (gi << 16));
                                wait_count(a.cnt + s.tile, nothers);
                                asm volatile("fence.proxy.async.global;" ::: "memory");
                                trace_point(110, blockIdx.x | (gi << 16));
                            }
                            const int t0 = jn * cap, nt = min(cap, T - t0);
                            if (!staged) {
                                ptx::mbar_arrive_expect_tx(&red_full[b2], 0);
                                return;
                            }
                            ptx::mbar_arrive_expect_tx(&red_full[b2], (uint32_t)((nothers + extra) * nt * kBM * 4));
                            uint8_t* dstb = b_base + b2 * stg_half;
                            for (int c = 0; c < nothers; ++c)
                                ptx::bulk_load(dstb + (size_t)c * cap * kBM * 4,
                                               a.part + ((size_t)s.tile * a.max_contrib + 1 + c) * kSlot + (size_t)t0 * kBM,
                                               (uint32_t)(nt * kBM * 4), &red_full[b2], pol_part);
                            if (extra)
                                for (int i = 0; i < nt; ++i)
                                    ptx::bulk_load(dstb + ((size_t)nothers * cap + i) * kBM * 4,
                                                   a.out_f32 + (size_t)(t0 + i) * a.ld_out + (size_t)s.tile * kBM,
                                                   kBM * 4, &red_full[b2], pol_part);
                        };
                        if (etid == 0) {
                            issue(0);
                            issue(1);
                        }
                        // warp 4's other lanes must not spin on the staging barrier while
                        // lane 0 is still issuing (a suspended spinning warp starves it)
                        __syncwarp();
                        for (int jn = 0; jn < njobs; ++jn) {
                            const int b2 = jn & 1;
                            ptx::mbar_wait(&red_full[b2], red_ph[b2]);
                            red_ph[b2] ^= 1u;
                            if (etid == 0) trace_point(107, blockIdx.x | (gi << 16) | (jn << 24));
                            const int t0 = jn * cap, nt = min(cap, T - t0);
                            const float* sm = (const float*)(b_base + b2 * stg_half);  // [c][cap tok][row]
                            const float* gp = a.part + (size_t)s.tile * a.max_contrib * kSlot + row;
                            const int nch = (nt + 15) / 16;
                            // both halves run the same number of chunks (argmax barriers pair up)
                            for (int jj = half; jj < nch + (nch & 1); jj += 2) {
                                const int tt = t0 + jj * 16;
                                float v[16];
                                if (jj < nch) {
                                    ptx::tmem_ld16(trow + tt, v);
                                    for (int c = 0; c < nothers; ++c) {
#pragma unroll
                                        for (int i = 0; i < 16; ++i) {
                                            if (jj * 16 + i >= nt) break;
                                            v[i] += staged ? sm[((size_t)c * cap + jj * 16 + i) * kBM + row]
                                                           : __ldcg(gp + (size_t)(1 + c) * kSlot + (size_t)(tt + i) * kBM);
                                        }
                                    }
                                    out16(tt, v, staged && extra ? sm + ((size_t)nothers * cap + jj * 16) * kBM + row
                                                                 : nullptr);
                                } else if (a.epi == EPI_ARGMAX) {
#pragma unroll
                                    for (int i = 0; i < 16; ++i) v[i] = -INFINITY;
                                    out16(T, v, nullptr);  // no tokens: barrier pairing only
                                }
                            }
                            ptx::named_bar_sync(1, kEpiThreads);  // staging buffer consumed
                            if (etid == 0) {
                                trace_point(108, blockIdx.x | (gi << 16) | (jn << 24));
                                issue(jn + 2);
                            }
                            __syncwarp();
                        }
                    }
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&tmem_empty[buf]);
                }
                if (etid == 0) trace_point(104, blockIdx.x | (gi << 16));
                if (a.epi < 0) continue;
                ptx::named_bar_sync(1, kEpiThreads);  // this CTA's owned tiles are written
                if (!a.owner_mode) {
                // ------------------------------------ reduction + epilogue of GEMM gi
                    // Jobs = (tile slice, token chunk).  Each job's nc contributor
                    // chunks are contiguous in the partial buffer ([slot][token][row])
                    // and are bulk-copied into the B ring -- idle until every CTA
                    // has finished this GEMM -- two jobs in flight, so the L2
                    // latency is paid once per job, not once per load.
                    {
                        const uint64_t pol_part = ptx::policy_evict_first();  // partials: read once
                        // this CTA's share of the GEMM's (tile, token) outputs
                        const long long W = (long long)a.m_tiles * T;
                        long long ix = (long long)blockIdx.x * W / G;
                        const long long ix_end = (long long)(blockIdx.x + 1) * W / G;
                        int prev_tile = -1;
                        RJob q[2];
                        auto issue = [&](int buf) {  // etid 0 only: next job into staging buffer `buf`
                            RJob j;
                            if (!rjob_next(r, ix, ix_end, prev_tile, j, G, T, stg_half, extra, P.dbg)) {
                                q[buf].nt = 0;
                                return;
                            }
                            q[buf] = j;
                            if (j.first) {
                                wait_count(a.cnt + j.tile, j.nc);
                                asm volatile("fence.proxy.async.global;" ::: "memory");
                            }
                            const uint32_t bytes = j.staged ? (uint32_t)((j.nc + extra) * j.nt * kBM * 4) : 0u;
                            ptx::mbar_arrive_expect_tx(&red_full[buf], bytes);
                            if (j.staged) {
                                uint8_t* dst = b_base + buf * stg_half;
                                for (int c = 0; c < j.nc; ++c)
                                    ptx::bulk_load(dst + (size_t)c * j.nt * kBM * 4,
                                                   a.part + ((size_t)j.tile * a.max_contrib + c) * kSlot + (size_t)j.t0 * kBM,
                                                   (uint32_t)(j.nt * kBM * 4), &red_full[buf], pol_part);
                                if (extra)  // this tile's 128 residual columns of each token
                                    for (int i = 0; i < j.nt; ++i)
                                        ptx::bulk_load(dst + ((size_t)j.nc * j.nt + i) * kBM * 4,
                                                       a.out_f32 + (size_t)(j.t0 + i) * a.ld_out + (size_t)j.tile * kBM,
                                                       kBM * 4, &red_full[buf], pol_part);
                            }
                        };
                        if (etid == 0) {
                            issue(0);
                            issue(1);
                            s_job[0] = q[0];
                            s_job[1] = q[1];
                        }
                        ptx::named_bar_sync(1, kEpiThreads);
                        for (int jn = 0;; ++jn) {
                            const int buf = jn & 1;
                            const RJob j = s_job[buf];
                            if (j.nt == 0) break;
                            ptx::mbar_wait(&red_full[buf], red_ph[buf]);
                            red_ph[buf] ^= 1u;
                            if (etid == 0) trace_point(107, blockIdx.x | (gi << 16) | (jn << 24));
                            float* sm = (float*)(b_base + buf * stg_half);  // [c][tok][row]
                            if (a.epi == EPI_ARGMAX) {
                                // sums back into contributor 0's chunk, then (max, lowest id) over
                                // the tile's rows per token: 4 threads per token, 32 rows each
                                // (skewed: no bank conflicts)
                                for (int i = half; i < j.nt; i += 2) {
                                    float v = 0.0f;
                                    for (int c = 0; c < j.nc; ++c) v += sm[((size_t)c * j.nt + i) * kBM + row];
                                    sm[(size_t)i * kBM + row] = v;
                                }
                                ptx::named_bar_sync(1, kEpiThreads);
                                bool bad = false;
                                for (int i0 = 0; i0 < j.nt; i0 += kEpiThreads / 4) {
                                    const int i = i0 + etid / 4, qq = etid % 4;
                                    float bv = -INFINITY;
                                    int bi = 0x7fffffff;
                                    if (i < j.nt) {
                                        for (int k = 0; k < 32; ++k) {
                                            const int rr = qq * 32 + ((k + i) & 31);
                                            const int mm = j.tile * kBM + rr;
                                            const float v = sm[(size_t)i * kBM + rr];
                                            if (mm < a.vocab) {
                                                if (a.logits) a.logits[(size_t)(j.t0 + i) * a.vocab + mm] = v;
                                                if (!isfinite(v)) bad = true;
                                                if (arg_better(v, mm, bv, bi)) {
                                                    bv = v;
                                                    bi = mm;
                                                }
                                            }
                                        }
                                    }
    #pragma unroll
                                    for (int off = 1; off < 4; off <<= 1) {
                                        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                                        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                                        if (arg_better(ov, oi, bv, bi)) {
                                            bv = ov;
                                            bi = oi;
                                        }
                                    }
                                    if (qq == 0 && i < j.nt) {
                                        const int t = j.t0 + i;
                                        a.arg_v[(size_t)t * kGemmMaxTiles + j.tile] = bv;
                                        a.arg_i[(size_t)t * kGemmMaxTiles + j.tile] = bi;
                                        __threadfence();
                                        if (atomicAdd(a.cnt + kTokCnt + t, 1) == a.m_tiles - 1)
                                            s_last[atomicAdd(&s_nlast, 1)] = t;
                                    }
                                }
                                if (bad) atomicExch(a.flag, 1);
                            } else {
                                // thread = 2 adjacent rows (float2 / bf16x2 accesses) x tokens
                                // q4, q4 + 4, ... of the job, two tokens in flight
                                const int r2 = (etid & 63) * 2, q4 = etid >> 6;
                                const int m2 = j.tile * kBM + r2;
                                if (m2 < a.M) {  // M is even: both rows valid
                                    const float2 bias = a.bias ? __ldg((const float2*)(a.bias + m2)) : make_float2(0.f, 0.f);
                                    // per-thread constants of the QKV scatter (the row pair fixes Q/K/V, head, d)
                                    int which = 0, hm = m2;
                                    size_t kv_base = 0, kv_sample = 0;
                                    if (a.epi == EPI_QKV) {
                                        which = m2 / a.h;
                                        hm = m2 - which * a.h;
                                        const int head = hm / a.hd, d = hm - head * a.hd;
                                        kv_sample = (size_t)a.heads * a.cap * a.hd;
                                        kv_base = ((size_t)a.layer * 2 + (which > 0 ? which - 1 : 0)) * a.B * kv_sample +
                                                  (size_t)head * a.cap * a.hd + d;
                                    }
                                    const float* gp2 = a.part + (size_t)j.tile * a.max_contrib * kSlot + r2;
                                    for (int i0 = q4; i0 < j.nt; i0 += 8) {
                                        float2 v[2];
    #pragma unroll
                                        for (int k = 0; k < 2; ++k) {
                                            const int i = i0 + 4 * k;
                                            v[k] = bias;
                                            if (i < j.nt) {
                                                if (j.staged) {
    #pragma unroll 4
                                                    for (int c = 0; c < j.nc; ++c) {
                                                        const float2 x = *(const float2*)(sm + ((size_t)c * j.nt + i) * kBM + r2);
                                                        v[k].x += x.x;
                                                        v[k].y += x.y;
                                                    }
                                                } else {
                                                    for (int c = 0; c < j.nc; ++c) {
                                                        const float2 x = __ldcg((const float2*)(gp2 + c * kSlot + (size_t)(j.t0 + i) * kBM));
                                                        v[k].x += x.x;
                                                        v[k].y += x.y;
                                                    }
                                                }
                                            }
                                        }
    #pragma unroll
                                        for (int k = 0; k < 2; ++k) {
                                            const int i = i0 + 4 * k;
                                            if (i >= j.nt) break;
                                            const int t = j.t0 + i;
                                            if (a.epi == EPI_RESID_LN) {
                                                float2* rp = (float2*)(a.out_f32 + (size_t)t * a.ld_out + m2);
                                                const float2 rv = j.staged ? *(const float2*)(sm + ((size_t)j.nc * j.nt + i) * kBM + r2)
                                                                           : __ldcg(rp);
                                                *rp = make_float2(rv.x + v[k].x, rv.y + v[k].y);
                                            } else if (a.epi == EPI_GELU) {
                                                *(__nv_bfloat162*)(a.out_bf16 + (size_t)t * a.ld_out + m2) =
                                                    __floats2bfloat162_rn(gelu_fast(v[k].x), gelu_fast(v[k].y));
                                            } else if (a.epi == EPI_QKV) {
                                                const __nv_bfloat162 x2 = __floats2bfloat162_rn(v[k].x, v[k].y);
                                                if (which == 0) {
                                                    *(__nv_bfloat162*)(a.out_bf16 + (size_t)t * a.h + hm) = x2;
                                                } else {
                                                    const Plan pl = a.plans[t];
                                                    if (pl.store)
                                                        *(__nv_bfloat162*)(a.kv + kv_base + (size_t)pl.sample * kv_sample +
                                                                           (size_t)pl.write_slot * a.hd) = x2;
                                                }
                                            } else {
                                                *(float2*)(a.out_f32 + (size_t)t * a.ld_out + m2) = v[k];
                                            }
                                        }
                                    }
                                }
                            }
                            ptx::named_bar_sync(1, kEpiThreads);  // staging buffer consumed
                            if (etid == 0) trace_point(108, blockIdx.x | (gi << 16) | (jn << 24));
                            if (etid == 0) {
                                issue(buf);
                                s_job[buf] = q[buf];
                            }
                            ptx::named_bar_sync(1, kEpiThreads);
                        }
                    }
    
                }
                if (etid == 0) trace_point(105, blockIdx.x | (gi << 16));
                if (a.epi == EPI_RESID_LN) {
                    // every tile's residual is final: LayerNorm rows blockIdx.x, +G, ...
                    if (etid == 0) {
                        __threadfence();
                        atomicAdd(a.cnt + kLnCnt, 1);
                        wait_count(a.cnt + kLnCnt, (int)G);
                    }
                    ptx::named_bar_sync(1, kEpiThreads);
                    for (int t = blockIdx.x; t < T; t += (int)G) ln_row(a, t, s_red);
                } else if (a.epi == EPI_ARGMAX) {
                    // tokens whose last vocab tile this CTA wrote: fold the per-tile partials
                    __threadfence();
                    for (int jj = warp - 4; jj < s_nlast; jj += kEpiThreads / 32) {
                        const int t = s_last[jj];
                        float bv = -INFINITY;
                        int bi = 0x7fffffff;
                        for (int tile = lane; tile < a.m_tiles; tile += 32) {
                            const float v = __ldcg(a.arg_v + (size_t)t * kGemmMaxTiles + tile);
                            const int id = __ldcg(a.arg_i + (size_t)t * kGemmMaxTiles + tile);
                            if (arg_better(v, id, bv, bi)) {
                                bv = v;
                                bi = id;
                            }
                        }
#pragma unroll
                        for (int off = 16; off > 0; off >>= 1) {
                            const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                            if (arg_better(ov, oi, bv, bi)) {
                                bv = ov;
                                bi = oi;
                            }
                        }
                        if (lane == 0) a.argmax[t] = bi == 0x7fffffff ? 0 : bi;
                    }
                }
                // this CTA is done with GEMM gi (outputs visible before the count)
                ptx::named_bar_sync(1, kEpiThreads);
                if (etid == 0) trace_point(106, blockIdx.x | (gi << 16));
                if (etid == 0 && gi + 1 < P.n) {
                    __threadfence();
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    atomicAdd(a.cnt + kDoneCnt, 1);
                }
            }
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

void plan_counts(int m_tiles, int KB, int G, int& max_contrib, int& n_slices) {
    long long U = (long long)m_tiles * KB;
    max_contrib = 1;
    n_slices = 0;
    for (int t = 0; t < m_tiles; ++t) {
        long long tk0 = (long long)t * KB;
        const int nc = U < G ? KB : cta_of(tk0 + KB - 1, G, U) - cta_of(tk0, G, U) + 1;
        max_contrib = std::max(max_contrib, nc);
        n_slices += nc;
    }
}

int g_sms = 148;  // grid of every chain launch (one CTA per SM)

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
    SD_CHECK(a.m_tiles >= 1 && a.m_tiles <= kGemmMaxTiles, CONFIG, "GEMM has too many 128-row tiles");
    plan_counts(a.m_tiles, a.K / kBK, sms, a.max_contrib, a.n_slices);
    // owner reduction keeps the owner's accumulator on chip and overlaps the
    // early contributors with the mainloop, but serialises a tile's whole
    // epilogue on one CTA: worth it only while tiles have few contributors
    static const int mode = getenv("SD_GEMM_OWNER") ? atoi(getenv("SD_GEMM_OWNER")) : -1;
    a.owner_mode = mode >= 0 ? mode : (a.max_contrib <= 3 ? 1 : 0);
}

size_t gemm_part_floats(int M, int K, int sms) {
    GemmArgs a{};
    a.M = M;
    a.K = K;
    a.m_tiles = (M + kBM - 1) / kBM;
    gemm_plan(a, sms);
    return (size_t)a.m_tiles * a.max_contrib * kSlot;
}

void gemm_prepare() {
    static bool done = false;
    if (done) return;
    CUDA_OK(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    done = true;
}

void chain_launch(const GemmChain& c, const GemmMaps* const* maps, cudaStream_t st) {
    gemm_prepare();
    SD_CHECK(c.n >= 1 && c.n <= kMaxChain, INTERNAL, "bad GEMM chain length");
    SD_CHECK(c.T_upper >= 1 && c.T_upper <= 256, INTERNAL, "GEMM token tile is 1..256");
    ChainParams p;
    std::memset(&p, 0, sizeof(p));
    p.n = c.n;
    p.T = c.T;
    p.dT = c.dT;
    p.box = c.T_upper <= 32 ? 32 : c.T_upper <= 64 ? 64 : c.T_upper <= 128 ? 128 : 256;
    const int bi = p.box == 32 ? 0 : p.box == 64 ? 1 : p.box == 128 ? 2 : 3;
    p.sb = c.sb;
    p.dbg = c.dbg;
    p.prefetch = c.prefetch;
    for (int i = 0; i < c.n; ++i) {
        const GemmArgs& a = c.g[i];
        SD_CHECK(a.cnt || a.epi < 0, INTERNAL, "GEMM call site has no counters");
        SD_CHECK(a.M % 2 == 0, CONFIG, "GEMM output features must be even (paired epilogue stores)");
        SD_CHECK(a.epi != EPI_RESID_LN || (a.M % 4 == 0 && a.M <= 8192), CONFIG,
                 "bf16 mode needs hidden % 4 == 0 and <= 8192");
        SD_CHECK(a.epi != EPI_ARGMAX || (a.arg_v && a.arg_i), INTERNAL, "argmax scratch missing");
        SD_CHECK(a.epi != EPI_ARGMAX || a.max_contrib * kBM * 4 <= 24576, INTERNAL,
                 "argmax tiles need their contributor rows to fit one staging buffer");
        SD_CHECK(i == 0 || a.part != c.g[i - 1].part, INTERNAL, "chained GEMMs need alternating partial buffers");
        p.g[i] = a;
        p.A[i] = maps[i]->A;
        p.B[i] = maps[i]->B[bi];
    }
    launch_k(k_gemm, dim3(g_sms), dim3(kThreads), kSmemBytes, st, p);
    CUDA_OK(cudaGetLastError());
}

}  // namespace sdb

// --------------------------------------------------------------- test hook
namespace {
thread_local std::string g_dbg_err;
}
extern "C" int sd_debug_gemm(const uint16_t* W, const uint16_t* X, int M, int K, int T, int grid, int flags,
                             float* Y, float* usec) {
    using namespace sdb;
    try {
        const int m_tiles = (M + kBM - 1) / kBM;
        const int sms = grid > 0 ? grid : 148;
        size_t wbytes = (size_t)m_tiles * kBM * K * 2, xbytes = (size_t)T * K * 2;
        void *dW = dmalloc(wbytes), *dX = dmalloc(xbytes), *dY = dmalloc((size_t)T * M * 4);
        int* dcnt = (int*)dmalloc(sizeof(int) * kGemmCntInts);
        GemmChain c{};
        c.n = 1;
        c.T = T;
        c.T_upper = T;
        c.sb = (flags >> 5) & 7;   // bits 5-7: token-ring depth (0 = default)
        c.dbg = (flags >> 1) & 3;  // bit1 skip MMAs, bit2 skip partial stores
        GemmArgs& a = c.g[0];
        a.epi = (flags & 8) ? -1 : EPI_STORE;  // bit3: time the streaming kernel alone
        a.M = M;
        a.K = K;
        a.m_tiles = m_tiles;
        gemm_plan(a, sms);
        void* dpart = dmalloc(sizeof(float) * (size_t)m_tiles * a.max_contrib * kSlot);
        CUDA_OK(cudaMemset(dW, 0, wbytes));
        CUDA_OK(cudaMemcpy(dW, W, (size_t)M * K * 2, cudaMemcpyHostToDevice));
        CUDA_OK(cudaMemcpy(dX, X, xbytes, cudaMemcpyHostToDevice));
        GemmMaps maps;
        maps.A = make_tmap_2d(dW, (int64_t)m_tiles * kBM, K, kBM);
        make_b_maps(maps, dX, T, K);
        const GemmMaps* mp[1] = {&maps};
        a.part = (float*)dpart;
        a.cnt = dcnt;
        a.out_f32 = (float*)dY;
        a.ld_out = M;
        const int saved = g_sms;
        g_sms = sms;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        CUDA_OK(cudaMemset(dcnt, 0, sizeof(int) * kGemmCntInts));
        chain_launch(c, mp, 0);  // warm-up / configure
        CUDA_OK(cudaMemset(dcnt, 0, sizeof(int) * kGemmCntInts));
        CUDA_OK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        chain_launch(c, mp, 0);
        cudaEventRecord(e1);
        CUDA_OK(cudaDeviceSynchronize());
        g_sms = saved;
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (usec) *usec = ms * 1000.0f;
        CUDA_OK(cudaMemcpy(Y, dY, (size_t)T * M * 4, cudaMemcpyDeviceToHost));
        dfree(dW);
        dfree(dX);
        dfree(dY);
        dfree(dpart);
        dfree(dcnt);
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
void trace_set_attn(const TraceBuf& b);
void trace_set_attn1(const TraceBuf& b);
}  // namespace sdb
namespace {
sdb::TraceBuf g_host_trace{nullptr, nullptr, 0};
}
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
        trace_set_gemm(g_host_trace);
        trace_set_fast(g_host_trace);
        trace_set_step(g_host_trace);
        trace_set_attn(g_host_trace);
        trace_set_attn1(g_host_trace);
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
        TraceBuf off{nullptr, nullptr, 0};
        trace_set_gemm(off);
        trace_set_fast(off);
        trace_set_step(off);
        trace_set_attn(off);
        trace_set_attn1(off);
        return 0;
    } catch (const Error& e) {
        g_dbg_err = e.what();
        return e.code;
    }
}

// --------------------------------------------------------------- chain test hook
// Two chained GEMMs in one persistent launch:
//   G1: H[T][M1] = X[T][K] . W1^T  with epilogue `epi1`:
//         EPI_GELU      -> act = bf16(gelu(H + b1))
//         EPI_RESID_LN  -> resid += H + b1; act = bf16(LayerNorm(resid)) (gain 1, bias 0)
//   G2: Y[T][M2] = act . W2^T + b2   (EPI_STORE, fp32)
// Returns Y, the final residual (RESID_LN) and act (as raw bf16 bits).
extern "C" int sd_debug_chain(const uint16_t* X, const uint16_t* W1, const float* b1, const uint16_t* W2,
                              const float* b2, float* resid, int T, int K, int M1, int M2, int epi1, int flags,
                              uint16_t* act_out, float* Y) {
    using namespace sdb;
    try {
        const int t1 = (M1 + kBM - 1) / kBM, t2 = (M2 + kBM - 1) / kBM;
        auto up = [](const void* h, size_t n) {
            void* d = dmalloc(n);
            CUDA_OK(cudaMemcpy(d, h, n, cudaMemcpyHostToDevice));
            return d;
        };
        void* dX = dmalloc((size_t)256 * K * 2);
        CUDA_OK(cudaMemset(dX, 0, (size_t)256 * K * 2));
        CUDA_OK(cudaMemcpy(dX, X, (size_t)T * K * 2, cudaMemcpyHostToDevice));
        void* dW1 = dmalloc((size_t)t1 * kBM * K * 2);
        CUDA_OK(cudaMemset(dW1, 0, (size_t)t1 * kBM * K * 2));
        CUDA_OK(cudaMemcpy(dW1, W1, (size_t)M1 * K * 2, cudaMemcpyHostToDevice));
        void* dW2 = dmalloc((size_t)t2 * kBM * M1 * 2);
        CUDA_OK(cudaMemset(dW2, 0, (size_t)t2 * kBM * M1 * 2));
        CUDA_OK(cudaMemcpy(dW2, W2, (size_t)M2 * M1 * 2, cudaMemcpyHostToDevice));
        void* db1 = up(b1, sizeof(float) * M1);
        void* db2 = up(b2, sizeof(float) * M2);
        void* dres = up(resid, sizeof(float) * (size_t)T * M1);
        std::vector<float> ones(M1, 1.0f), zeros(M1, 0.0f);
        void* dg = up(ones.data(), sizeof(float) * M1);
        void* dbz = up(zeros.data(), sizeof(float) * M1);
        void* dact = dmalloc((size_t)256 * M1 * 2);
        CUDA_OK(cudaMemset(dact, 0, (size_t)256 * M1 * 2));
        void* dY = dmalloc(sizeof(float) * (size_t)T * M2);
        int* dcnt = (int*)dmalloc(sizeof(int) * 2 * kGemmCntInts);
        CUDA_OK(cudaMemset(dcnt, 0, sizeof(int) * 2 * kGemmCntInts));
        GemmChain c{};
        c.n = 2;
        c.T = T;
        c.T_upper = T;
        c.dbg = flags;
        GemmArgs& a = c.g[0];
        a.epi = epi1;
        a.M = M1;
        a.K = K;
        a.m_tiles = t1;
        gemm_plan(a, g_sms);
        a.cnt = dcnt;
        a.bias = (const float*)db1;
        if (epi1 == EPI_GELU) {
            a.out_bf16 = (__nv_bfloat16*)dact;
            a.ld_out = M1;
        } else {
            a.out_f32 = (float*)dres;
            a.ld_out = M1;
            a.ln_g = (const float*)dg;
            a.ln_b = (const float*)dbz;
            a.ln_out = (__nv_bfloat16*)dact;
        }
        GemmArgs& b = c.g[1];
        b.epi = EPI_STORE;
        b.M = M2;
        b.K = M1;
        b.m_tiles = t2;
        gemm_plan(b, g_sms);
        b.cnt = dcnt + kGemmCntInts;
        b.bias = (const float*)db2;
        b.out_f32 = (float*)dY;
        b.ld_out = M2;
        void* p1 = dmalloc(sizeof(float) * (size_t)t1 * a.max_contrib * kSlot);
        void* p2 = dmalloc(sizeof(float) * (size_t)t2 * b.max_contrib * kSlot);
        a.part = (float*)p1;
        b.part = (float*)p2;
        GemmMaps m1, m2;
        m1.A = make_tmap_2d(dW1, (int64_t)t1 * kBM, K, kBM);
        make_b_maps(m1, dX, 256, K);
        m2.A = make_tmap_2d(dW2, (int64_t)t2 * kBM, M1, kBM);
        make_b_maps(m2, dact, 256, M1);
        const GemmMaps* mp[2] = {&m1, &m2};
        chain_launch(c, mp, 0);
        CUDA_OK(cudaDeviceSynchronize());
        CUDA_OK(cudaMemcpy(Y, dY, sizeof(float) * (size_t)T * M2, cudaMemcpyDeviceToHost));
        CUDA_OK(cudaMemcpy(act_out, dact, (size_t)T * M1 * 2, cudaMemcpyDeviceToHost));
        CUDA_OK(cudaMemcpy(resid, dres, sizeof(float) * (size_t)T * M1, cudaMemcpyDeviceToHost));
        for (void* p : {dX, dW1, dW2, db1, db2, dres, dg, dbz, dact, dY, (void*)dcnt, p1, p2}) dfree(p);
        return 0;
    } catch (const Error& e) {
        g_dbg_err = e.what();
        return e.code;
    }
}
