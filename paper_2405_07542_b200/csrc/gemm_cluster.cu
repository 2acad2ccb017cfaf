// Cluster split-K tcgen05 GEMM for small models (hidden <= 1024, e.g. the
// OPT-125m-shaped C2 target and the C4 draft).
//
//   Y[t][m] = sum_k W[m][k] * X[t][k]       (W = weights [M][K], X = tokens [T][K])
//
// At these sizes a verify step is a chain of latency-bound launches, not a
// bandwidth problem (C2 streams ~0.4 GB per step): the stream-K GEMM of
// gemm_sm100.cu spends more on its separate split-K reduction and LayerNorm
// launches than on the weights.  Here one launch does the whole GEMM stage:
//
//   * a 128-row weight tile is split over the CS CTAs of one thread-block
//     cluster along K (CS <= 16, each CTA holds its whole k-range in shared
//     memory: no ring), every CTA issuing tcgen05.mma into its own TMEM
//     accumulator (M = 128 rows, N = the packed tokens);
//   * the CS fp32 partial tiles are summed inside the cluster through
//     distributed shared memory in fixed rank order (deterministic, no global
//     partials): CTA r owns a contiguous run of tokens, every CTA pushes its
//     rows of that run into r's shared memory with one bulk copy
//     (cp.async.bulk shared::cta -> shared::cluster, completing on r's
//     mbarrier), r sums them one warp per token;
//   * the epilogue is fused: bias + Q/K/V scatter into the unpadded KV arena,
//     bias + GELU, or bias + residual update plus the per-(token, 128-row tile)
//     LayerNorm statistics (sum, M2) of the new residual rows;
//   * the NEXT GEMM applies that LayerNorm while it builds its token operand
//     (LN_IN): per-token mean / rstd Chan-combined from the tile statistics in
//     fixed order, (x - mean) * rstd * gamma + beta packed to bf16 straight
//     into the 128B-swizzled K-major layout the MMA reads.
//
// A transformer layer is therefore QKV -> attention -> O -> FC -> PROJ: five
// launches instead of eleven.  The split (CS, k-range per CTA) depends only on
// the GEMM shape and the SM count, never on the token count, so a token's
// result does not depend on the batch it is verified in.
//
// One launch covers at most 128 tokens (a 256-token forward chunk is two
// launches per GEMM over token halves, t_base = 0 / 128: the weights of a
// small model stay in L2 between them).
//
// At most half the SMs per launch (so a launch and its PDL-overlapped
// successor fit side by side, one CTA per SM); C2: QKV 18 tiles x CS 4, O 6 x
// 12, FC 24 x 3, PROJ 6 x 12.
//
// Warp roles (256 threads): thread 0 TMA (weights before griddepcontrol.wait,
// tokens after, fetched with the token count in one round trip), warp 1 TMEM
// allocation + lane 0 MMA issue, warps 4-7 copy their TMEM rows to shared
// memory and lane r of warp 4 ships owner r's run with one bulk copy, all 8
// warps the LN_IN operand build and the owner-side reduction + epilogue.  A
// relaxed cluster barrier at entry (barrier inits visible) and an
// arrive (all incoming copies landed) / wait (before exit) pair are the only
// cluster-wide synchronisation.
#include <cuda_bf16.h>

#include <algorithm>

#include "gemm.h"
#include "pdl.cuh"
#include "sm100_ptx.cuh"
#include "trace.cuh"

SD_TRACE_TU(gemmcl)

namespace sdb {
namespace {

constexpr int kClThreads = 256;
constexpr int kClABytes = 128 * 64 * 2;  // one 128-row x 64-k bf16 weight block (16 KB)
constexpr int kClMaxKb = 4;              // k-blocks per CTA (whole k-range resident)
constexpr int kClMaxCS = 16;
constexpr int kClSmemMax = 220 * 1024;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// execution-only cluster barrier (no memory fence: nothing is published
// through ordinary memory; barrier inits are covered by
// fence.mbarrier_init.release.cluster, the bulk copies by their mbarriers)
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
// bulk copy of this CTA's shared memory into a peer's (both shared::cluster
// addresses), completing on the peer's mbarrier
__device__ __forceinline__ void bulk_s2c(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "r"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tmem_alloc_n(uint32_t* dst, uint32_t cols) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(dst)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc_n(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float gelu_tanh(float x) {  // model.cpp:71-74, hardware tanh
    const float c = 0.7978845608028654f;
    float u = c * (x + 0.044715f * x * x * x);
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
    return 0.5f * x * (1.0f + t);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

template <int EPI, bool LN_IN>
__global__ void __launch_bounds__(kClThreads, 1)
    k_gemm_cl(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB32,
              const __grid_constant__ CUtensorMap tmB64, const __grid_constant__ CUtensorMap tmB128,
              const ClArgs a) {
    CtaTrace trace__(EPI == EPI_QKV ? TK_GEMM_CL_QKV : EPI == EPI_GELU ? TK_GEMM_CL_GELU : TK_GEMM_CL_RESID);
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned by pointer arithmetic on the __shared__ array, so every
    // access below stays a shared-memory instruction (no generic ST/LD)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t s_full_a[kClMaxKb], s_full_b, s_tmem_full, s_recv;
    __shared__ uint32_t s_tmem;
    __shared__ float4 s_g[kClMaxKb * 16], s_b[kClMaxKb * 16];  // LN gamma / beta of this CTA's k-range
    __shared__ float s_mu[128], s_rs[128];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int CS = a.CS;
    const int rank = (int)cluster_rank();
    const int tile = blockIdx.x / CS;
    const int KB = a.K / 64;
    const int kb0 = rank * KB / CS, nkb = (rank + 1) * KB / CS - kb0;
    const int box = a.box;                          // host bound on this launch's tokens (<= 128)
    const int per_owner = a.per_owner;              // CTA r reduces tokens [r * per_owner, (r + 1) * per_owner)
    uint8_t* A = smem;                              // [nkb_max][128 rows][128 B]
    uint8_t* Bt = smem + a.nkb_max * kClABytes;     // [nkb_max][box rows][128 B]
    float* send = (float*)smem;                     // after the MMAs: [token][128 rows] fp32
    float* recv = (float*)(smem + a.recv_off);      // [sender][slot][128 rows] fp32

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmA);
        for (int i = 0; i < nkb; ++i) ptx::mbar_init(&s_full_a[i], 1);
        ptx::mbar_init(&s_full_b, 1);
        ptx::mbar_init(&s_tmem_full, 1);
        ptx::mbar_init(&s_recv, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_n(&s_tmem, (uint32_t)box);
    // everything that does not depend on the predecessor is issued before
    // griddepcontrol.wait: the weight blocks, LN gamma / beta, the bias
    if constexpr (LN_IN) {
        for (int i = threadIdx.x; i < nkb * 16; i += kClThreads) {
            s_g[i] = ((const float4*)(a.ln_g + kb0 * 64))[i];
            s_b[i] = ((const float4*)(a.ln_b + kb0 * 64))[i];
        }
    }
    ptx::tc_fence_before();
    __syncthreads();     // TMEM address, gamma / beta visible inside the CTA
    cluster_sync_all();  // barrier inits visible cluster-wide before any peer's bulk copy lands
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;
    pdl_trigger();
    if (threadIdx.x == 0) {
        const uint64_t pol_w = ptx::policy_evict_first();
        for (int i = 0; i < nkb; ++i) {
            ptx::mbar_arrive_expect_tx(&s_full_a[i], kClABytes);
            ptx::tma_load_2d(A + i * kClABytes, &tmA, &s_full_a[i], (kb0 + i) * 64, tile * 128, pol_w);
        }
    }
    const int m0 = tile * 128 + lane * 4;
    const float4 bias = a.bias ? *(const float4*)(a.bias + m0) : make_float4(0.f, 0.f, 0.f, 0.f);
    pdl_wait();
    // The token count and the token operand are fetched in the same round trip:
    // operand rows are read up to the host bound on this launch's tokens (rows
    // >= T are stale and never leave the CTA: the MMA uses N = BN, the owners
    // reduce only t < T)
    const int T_raw = a.dT ? *a.dT : a.T;
    constexpr int kU = 4;
    float4 xr[kU][2];
    float2 st[8];
    const int per_h = box * 8, total_h = nkb * per_h;  // 16-byte chunks of the LN_IN operand
    const int T_h = min(box, a.T - a.t_base);  // host bound on the rows that exist in this chunk
    const int i_0 = threadIdx.x / per_h, r_0 = threadIdx.x - i_0 * per_h;
    if constexpr (LN_IN) {
        // chunk idx = threadIdx.x + u * 256 -> (k-block i, token t, 16-byte chunk c),
        // advanced incrementally (no integer division in the loops)
        int ci = i_0, cr = r_0;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int idx = threadIdx.x + u * kClThreads;
            const int i = ci, t = cr >> 3, c = cr & 7;
            cr += kClThreads;
            while (cr >= per_h) {
                cr -= per_h;
                ++ci;
            }
            if (idx < total_h && t < T_h) {
                const float4* x = (const float4*)(a.x_resid + (size_t)(a.t_base + t) * a.hidden + (kb0 + i) * 64 + c * 8);
                xr[u][0] = x[0];
                xr[u][1] = x[1];
            }
        }
        if (threadIdx.x < T_h) {
            const float2* p = a.stats_in + (size_t)(a.t_base + threadIdx.x) * a.n_stat;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < a.n_stat) st[j] = p[j];
        }
    } else if (threadIdx.x == 0) {
        const CUtensorMap* tmB = box == 32 ? &tmB32 : box == 64 ? &tmB64 : &tmB128;
        const uint64_t pol_x = ptx::policy_evict_last();
        ptx::mbar_arrive_expect_tx(&s_full_b, (uint32_t)(nkb * box * 128));
        for (int i = 0; i < nkb; ++i)
            ptx::tma_load_2d(Bt + i * box * 128, tmB, &s_full_b, (kb0 + i) * 64, a.t_base, pol_x);
    }
    const int T = min(max(T_raw - a.t_base, 0), box);  // this launch's tokens
    const int BN = T <= 16 ? 16 : ((T + 15) / 16) * 16;
    const bool idle = T <= 0;
    const int own0 = rank * per_owner;
    const int n_own = min(max(T - own0, 0), per_owner);  // tokens this CTA reduces
    if (threadIdx.x == 0) ptx::mbar_arrive_expect_tx(&s_recv, (uint32_t)(CS * n_own * 512));
    const uint32_t ttag = ((uint32_t)EPI << 24) | blockIdx.x;
    if (threadIdx.x == 0) trace__.point(120, ttag);
    // the epilogue operands of this warp's first token, in flight during the MMAs
    const int t_first = own0 + warp;  // warp w reduces slots w, w + 8, ...
    float4 pre_old = make_float4(0.f, 0.f, 0.f, 0.f);
    Plan pre_pl{};
    if (t_first < T) {
        if constexpr (EPI == EPI_RESID_LN) pre_old = *(const float4*)(a.resid + (size_t)(a.t_base + t_first) * a.hidden + m0);
        if constexpr (EPI == EPI_QKV) pre_pl = a.plans[a.t_base + t_first];
    }
    if (!idle) {
        if constexpr (LN_IN) {
            // LN(x) -> bf16 in the 128B-swizzled K-major layout TMA would
            // produce (16-byte chunk c of row t at chunk c ^ (t & 7)); per-token
            // statistics: Chan combination of the producer's per-tile (sum, M2)
            // in tile order (deterministic)
            if (threadIdx.x < T) {
                float sm = 0.0f;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < a.n_stat) sm += st[j].x;
                const float mu = sm / a.hidden;
                float m2 = 0.0f;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < a.n_stat) {
                        const float d = st[j].x * (1.0f / 128.0f) - mu;
                        m2 += st[j].y + 128.0f * d * d;
                    }
                s_mu[threadIdx.x] = mu;
                s_rs[threadIdx.x] = rsqrtf(m2 / a.hidden + 1e-5f);
            }
            __syncthreads();
            int ci = i_0, cr = r_0;
            for (int u0 = 0; u0 * kClThreads < total_h; u0 += kU) {
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const int idx = threadIdx.x + (u0 + u) * kClThreads;
                    if (idx >= total_h) break;
                    const int i = ci, t = cr >> 3, c = cr & 7;
                    cr += kClThreads;
                    while (cr >= per_h) {
                        cr -= per_h;
                        ++ci;
                    }
                    if (u0 > 0 && t < T) {  // chunks beyond the first four per thread (box * nkb > 128)
                        const float4* x = (const float4*)(a.x_resid + (size_t)(a.t_base + t) * a.hidden + (kb0 + i) * 64 + c * 8);
                        xr[u][0] = x[0];
                        xr[u][1] = x[1];
                    }
                    uint4 o = make_uint4(0u, 0u, 0u, 0u);
                    if (t < T) {
                        const float mu = s_mu[t], rs = s_rs[t];
                        const float4 x0 = xr[u][0], x1 = xr[u][1];
                        const float4 g0 = s_g[i * 16 + c * 2], g1 = s_g[i * 16 + c * 2 + 1];
                        const float4 b0 = s_b[i * 16 + c * 2], b1 = s_b[i * 16 + c * 2 + 1];
                        o.x = pack_bf16((x0.x - mu) * rs * g0.x + b0.x, (x0.y - mu) * rs * g0.y + b0.y);
                        o.y = pack_bf16((x0.z - mu) * rs * g0.z + b0.z, (x0.w - mu) * rs * g0.w + b0.w);
                        o.z = pack_bf16((x1.x - mu) * rs * g1.x + b1.x, (x1.y - mu) * rs * g1.y + b1.y);
                        o.w = pack_bf16((x1.z - mu) * rs * g1.z + b1.z, (x1.w - mu) * rs * g1.w + b1.w);
                    }
                    *(uint4*)(Bt + i * box * 128 + t * 128 + ((c ^ (t & 7)) << 4)) = o;
                }
            }
            ptx::fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
            __syncthreads();
            if (threadIdx.x == 0) trace__.point(121, ttag);
        }
        if (threadIdx.x == 32) {  // ---------------- MMA issuer
            const uint32_t idesc = ptx::umma_idesc_bf16(128, BN);
            if (!LN_IN) ptx::mbar_wait(&s_full_b, 0);
            for (int i = 0; i < nkb; ++i) {
                ptx::mbar_wait(&s_full_a[i], 0);
                ptx::tc_fence_after();
                const uint32_t sa = ptx::smem_u32(A + i * kClABytes), sb = ptx::smem_u32(Bt + i * box * 128);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    ptx::umma_bf16(tmem, ptx::umma_desc_kmajor_sw128(sa + k * 32), ptx::umma_desc_kmajor_sw128(sb + k * 32),
                                   idesc, (i > 0 || k > 0) ? 1u : 0u);
            }
            ptx::umma_commit(&s_tmem_full);
        }
        if (warp >= 4) {  // ---------------- TMEM -> send buffer -> bulk copies to the owners
            ptx::mbar_wait(&s_tmem_full, 0);
            ptx::tc_fence_after();
            if (threadIdx.x == 128) trace__.point(122, ttag);
            const int row = (warp - 4) * 32 + lane;
            const uint32_t trow = tmem + ((uint32_t)((warp - 4) * 32) << 16);
            for (int j0 = 0; j0 < BN; j0 += 16) {
                float v[16];
                ptx::tmem_ld16(trow + j0, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) send[(j0 + i) * 128 + row] = v[i];
            }
            if (threadIdx.x == 128) trace__.point(126, ttag);
            ptx::fence_proxy_async_smem();  // the bulk copies read what the generic proxy wrote
            ptx::named_bar_sync(1, 128);
            if (warp == 4) {  // lane r ships owner r's run (CS <= 32)
                if (lane == 0) trace__.point(127, ttag);
                const int r = lane;
                const int nr = r < CS ? min(max(T - r * per_owner, 0), per_owner) : 0;
                if (nr > 0) {
                    const uint32_t src = ptx::smem_u32(send + (size_t)r * per_owner * 128);
                    const uint32_t dst = mapa_u32(ptx::smem_u32(recv + (size_t)rank * per_owner * 128), (uint32_t)r);
                    const uint32_t bar = mapa_u32(ptx::smem_u32(&s_recv), (uint32_t)r);
                    bulk_s2c(dst, src, (uint32_t)(nr * 512), bar);
                }
                __syncwarp();
                if (lane == 0) trace__.point(123, ttag);
            }
        }
    } else if (threadIdx.x == 0) {  // no TMA in flight at exit
        for (int i = 0; i < nkb; ++i) ptx::mbar_wait(&s_full_a[i], 0);
        if (!LN_IN) ptx::mbar_wait(&s_full_b, 0);
    }
    ptx::mbar_wait(&s_recv, 0);  // every sender's rows of this CTA's tokens have landed
    __syncwarp();
    cluster_arrive();            // ... so this CTA's incoming copies are complete
    if (threadIdx.x == 0) trace__.point(124, ttag);
    int it = 0;
    for (int slot = warp; slot < n_own; slot += kClThreads / 32, ++it) {
        const int t = own0 + slot;
        float4 v[kClMaxCS];  // every sender's rows loaded before the first add
#pragma unroll
        for (int p = 0; p < kClMaxCS; ++p)
            if (p < CS) v[p] = *(const float4*)(recv + ((size_t)p * per_owner + slot) * 128 + lane * 4);
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int p = 0; p < kClMaxCS; ++p)  // fixed rank order: deterministic
            if (p < CS) {
                s.x += v[p].x;
                s.y += v[p].y;
                s.z += v[p].z;
                s.w += v[p].w;
            }
        const size_t tg = (size_t)(a.t_base + t);
        if constexpr (EPI == EPI_RESID_LN) {
            float4* rp = (float4*)(a.resid + tg * a.hidden + m0);
            const float4 o = it == 0 ? pre_old : *rp;
            const float4 x = make_float4(o.x + (s.x + bias.x), o.y + (s.y + bias.y), o.z + (s.z + bias.z),
                                         o.w + (s.w + bias.w));
            *rp = x;
            const float sum = warp_sum(x.x + x.y + x.z + x.w);
            const float mu = sum * (1.0f / 128.0f);
            const float dx = x.x - mu, dy = x.y - mu, dz = x.z - mu, dw = x.w - mu;
            const float m2 = warp_sum(dx * dx + dy * dy + dz * dz + dw * dw);
            if (lane == 0) a.stats_out[tg * a.n_stat + tile] = make_float2(sum, m2);
        } else if constexpr (EPI == EPI_GELU) {
            uint2 o;
            o.x = pack_bf16(gelu_tanh(s.x + bias.x), gelu_tanh(s.y + bias.y));
            o.y = pack_bf16(gelu_tanh(s.z + bias.z), gelu_tanh(s.w + bias.w));
            *(uint2*)(a.out_bf16 + tg * a.ld_out + m0) = o;
        } else {  // EPI_QKV
            uint2 o;
            o.x = pack_bf16(s.x + bias.x, s.y + bias.y);
            o.y = pack_bf16(s.z + bias.z, s.w + bias.w);
            const int which = m0 / a.h, hm = m0 - which * a.h;
            if (which == 0) {
                *(uint2*)(a.out_bf16 + tg * a.h + hm) = o;
            } else {
                const Plan pl = it == 0 ? pre_pl : a.plans[tg];
                if (pl.store) {
                    const int head = hm / a.hd, d = hm - head * a.hd;
                    const size_t off = ((((size_t)a.layer * 2 + (which - 1)) * a.B + pl.sample) * a.heads + head) *
                                           (size_t)a.cap * a.hd +
                                       (size_t)pl.write_slot * a.hd + d;
                    *(uint2*)(a.kv + off) = o;
                }
            }
        }
    }
    if (threadIdx.x == 0) trace__.point(125, ttag);
    __syncwarp();
    cluster_wait();  // every owner has received everything: no copy still reads this CTA's memory
    if (warp == 1) {
        ptx::tc_fence_after();
        tmem_dealloc_n(tmem, (uint32_t)box);
    }
}

template <int EPI, bool LN_IN>
void prepare_one() {
    auto k = k_gemm_cl<EPI, LN_IN>;
    CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kClSmemMax));
    CUDA_OK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

}  // namespace

ClPlan gemm_cl_plan(int M, int K, int box, int sms) {
    ClPlan p{};
    if (M % 128 || K % 64 || box < 32 || box > 128) return p;
    const int tiles = M / 128, KB = K / 64;
    // at most half the SMs, so a launch and its (PDL-overlapped) successor fit
    // side by side: one CTA per SM (shared memory), no second wave
    const int max_ctas = std::max(1, sms / 2);
    int cs = std::max((KB + kClMaxKb - 1) / kClMaxKb, std::min({kClMaxCS, max_ctas / std::max(1, tiles), KB}));
    if (cs < 1 || cs > kClMaxCS || cs > KB || (long long)tiles * cs > sms) return p;
    const int nkb = (KB + cs - 1) / cs;
    p.per_owner = (box + cs - 1) / cs;
    const size_t send = (size_t)box * 128 * 4;                     // [token][row] fp32
    const size_t recv = (size_t)cs * p.per_owner * 128 * 4;         // [sender][slot][row] fp32
    const size_t ab = (size_t)nkb * kClABytes + (size_t)nkb * box * 128;
    p.recv_off = (std::max(ab, send) + 1023) / 1024 * 1024;  // the send buffer reuses the operand tiles
    const size_t smem = p.recv_off + recv + 1024;
    if (smem > (size_t)kClSmemMax) return p;
    p.ok = true;
    p.CS = cs;
    p.nkb_max = nkb;
    p.tiles = tiles;
    p.smem = smem;
    return p;
}

void gemm_cl_prepare() {
    if (!first_use_on_device(3)) return;
    prepare_one<EPI_QKV, true>();
    prepare_one<EPI_GELU, true>();
    prepare_one<EPI_RESID_LN, false>();
}

bool gemm_cl_schedulable(const ClPlan& p) {
    gemm_cl_prepare();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.tiles * p.CS);
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = p.smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_gemm_cl<EPI_RESID_LN, false>, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return n >= 1;
}

void gemm_cl_launch(int epi, const ClArgs& a0, const GemmMaps& maps, int T_upper, cudaStream_t st) {
    gemm_cl_prepare();
    SD_CHECK(T_upper >= 1 && T_upper <= 128, INTERNAL, "cluster GEMM token tile is at most 128");
    ClArgs a = a0;
    a.box = T_upper <= 32 ? 32 : T_upper <= 64 ? 64 : 128;
    const ClPlan p = gemm_cl_plan(a.M, a.K, a.box, device_sm_count());
    SD_CHECK(p.ok, INTERNAL, "cluster GEMM plan infeasible for this shape");
    a.CS = p.CS;
    a.nkb_max = p.nkb_max;
    a.recv_off = (int)p.recv_off;
    a.per_owner = p.per_owner;
    const dim3 grid(p.tiles * p.CS);
    switch (epi) {
        case EPI_QKV:
            launch_kc(k_gemm_cl<EPI_QKV, true>, grid, dim3(kClThreads), p.smem, st, p.CS, maps.A, maps.B[0],
                      maps.B[1], maps.B[2], a);
            break;
        case EPI_GELU:
            launch_kc(k_gemm_cl<EPI_GELU, true>, grid, dim3(kClThreads), p.smem, st, p.CS, maps.A, maps.B[0],
                      maps.B[1], maps.B[2], a);
            break;
        case EPI_RESID_LN:
            launch_kc(k_gemm_cl<EPI_RESID_LN, false>, grid, dim3(kClThreads), p.smem, st, p.CS, maps.A, maps.B[0],
                      maps.B[1], maps.B[2], a);
            break;
        default:
            throw Error(INTERNAL, "cluster GEMM epilogue not supported");
    }
    CUDA_OK(cudaGetLastError());
}

}  // namespace sdb
