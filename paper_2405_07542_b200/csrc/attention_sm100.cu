// Ragged multi-query attention of the verify step (model.cpp:320-349 over
// UnpadArena::gather_visible, kv_cache.cpp:140-150), bf16 performance mode.
//
// The work is a list of items (sample, head, 8-query tile, 256-key split):
// each sample reads only ITS KV extent [0, kv_len) -- no pad tokens, no padded
// KV -- and each query additionally sees only slots <= its own write slot
// (causal within the drafts).  A persistent grid of one CTA per SM walks the
// item list round-robin with a warp-specialised pipeline:
//
//   warp 4      TMA producer: 64-key K and V chunks of every item, 128-byte
//               swizzled boxes, into a ring of kStages stages; it runs ahead
//               across item boundaries, so HBM never waits for the merge /
//               split-combine work of the compute warps.
//   warps 0-3   "keys as M" mma.sync (S^T = K Q^T, O^T += V^T P^T): each warp
//               owns 16 keys of a chunk and keeps an online softmax (running
//               max, sum, O^T) across the item's chunks; P^T is re-laid from
//               the S^T accumulators with movmatrix (no smem trip).  At the
//               end of an item the four warps merge through smem, and a split
//               either writes the context row (single split) or its partial;
//               the last split to arrive (per sample, head, query tile) folds
//               all partials in split order (deterministic) -- no combine kernel.
//
// With n_s <= 8 draft queries per sample a 16-query tile would be mostly
// padding, so keys are the 16-row M side and queries the 8-wide N side.  A
// sample's KV is read once per layer regardless of n_s (the paper's per-token
// grid, re-reads it n_s times).
#include <cuda_bf16.h>

#include <cstdlib>
#include <string>

#include "attn.h"
#include "gemm.h"
#include "pdl.cuh"
#include "sm100_ptx.cuh"
#include "trace.cuh"

SD_TRACE_TU(attn)

namespace sdb {
namespace {

constexpr int kComputeThreads = 128, kThreads = 160;

template <int HD, int STAGES>
struct ACfg {
    static constexpr int kHalfBytes = kAttnChunk * 128;               // one 64-column SW128 box
    static constexpr int kChunkBytes = kAttnChunk * HD * 2;           // K (or V) of one chunk
    static constexpr int kQBytes = kAttnQT * HD * 2;                  // one item's Q tile
    static constexpr int kQSlots = 4;                                 // items in flight (Q ring)
    static constexpr int kStageBytes = 2 * kChunkBytes;               // K + V
    static constexpr int kStages = STAGES;
    static constexpr int kRingBytes = kStages * kStageBytes;
    static constexpr int kSmem = 1024 + kRingBytes + kQSlots * kQBytes + 512;
};

// byte offset of (key row, hd col) inside a K or V chunk staged by TMA as
// HD/64 boxes of [64 rows][128 B] with the 128-byte swizzle
__device__ __forceinline__ uint32_t tswz(int row, int col) {
    return (uint32_t)((col >> 6) * (kAttnChunk * 128) + row * 128 + ((((col & 63) >> 3) ^ (row & 7)) << 4) +
                      ((col & 7) << 1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

struct Item {
    int s, head, qt, split, k_begin, k_end, nq, nsplit;
    bool valid;
};
__device__ __forceinline__ Item item_at(const AttnArgs& a, int i, int splits, int qtiles) {
    Item it;
    it.split = i % splits;
    const int rest = i / splits;
    it.qt = rest % qtiles;
    const int pair = rest / qtiles;
    it.s = pair / a.heads;
    it.head = pair - it.s * a.heads;
    const SampleSeg seg = a.segs[it.s];
    it.k_begin = it.split * kAttnSplit;
    it.k_end = min(seg.kv_len, it.k_begin + kAttnSplit);
    it.nq = min(kAttnQT, seg.n_q - it.qt * kAttnQT);
    it.nsplit = (seg.kv_len + kAttnSplit - 1) / kAttnSplit;
    it.valid = it.nq > 0 && it.k_begin < seg.kv_len;
    return it;
}

template <int HD, int STAGES, int CTAS>
__global__ void __launch_bounds__(kThreads, CTAS)
    k_attention(const __grid_constant__ CUtensorMap tm, const AttnArgs a, int splits, int qtiles) {
    CtaTrace trace__(TK_ATTN);
    using C = ACfg<HD, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* ring = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* qring = ring + C::kRingBytes;               // [kQSlots][8][HD] bf16
    uint64_t* full = (uint64_t*)(qring + C::kQSlots * C::kQBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* q_full = empty + C::kStages;
    uint64_t* q_empty = q_full + C::kQSlots;
    __shared__ int sq_item[C::kQSlots];  // item index of each Q slot (-1: no more work)

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int n_items = a.B * a.heads * qtiles * splits;
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tm);
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);  // released by the warp that processed the chunk
        }
        for (int s = 0; s < C::kQSlots; ++s) {
            ptx::mbar_init(&q_full[s], 1);
            ptx::mbar_init(&q_empty[s], 4);  // every compute warp loads the item's Q
        }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    pdl_trigger();
    pdl_wait();  // the packed batch descriptors, Q and this layer's K/V come from earlier kernels

    if (warp == 4) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();  // KV: streamed once per layer
            int stage = 0, qs = 0;
            uint32_t phase = 0, qph = 0;
            int next = atomicAdd(a.work, 1);  // dynamic: items have very different lengths
            for (;;) {
                const int i = next;
                if (i >= n_items) break;
                next = atomicAdd(a.work, 1);  // in flight while this item is issued
                const Item it = item_at(a, i, splits, qtiles);
                if (!it.valid) continue;
                const SampleSeg seg = a.segs[it.s];
                int toks[kAttnQT];  // rows past nq repeat row 0 (their outputs are unused)
#pragma unroll
                for (int r = 0; r < kAttnQT; ++r) toks[r] = a.qidx[seg.q_start + it.qt * kAttnQT + (r < it.nq ? r : 0)];
                ptx::mbar_wait(&q_empty[qs], qph ^ 1);
                sq_item[qs] = i;  // published by the arrive below
                ptx::mbar_arrive_expect_tx(&q_full[qs], C::kQBytes);
#pragma unroll
                for (int r = 0; r < kAttnQT; ++r)
                    ptx::bulk_load(qring + qs * C::kQBytes + r * HD * 2, a.q + (size_t)toks[r] * a.h + it.head * HD,
                                   HD * 2, &q_full[qs], pol);
                if (++qs == C::kQSlots) {
                    qs = 0;
                    qph ^= 1;
                }
                const int rk = ((((a.layer * 2 + 0) * a.B + it.s) * a.heads + it.head) * a.cap);
                const int rv = ((((a.layer * 2 + 1) * a.B + it.s) * a.heads + it.head) * a.cap);
                for (int k0 = it.k_begin; k0 < it.k_end; k0 += kAttnChunk) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                    uint8_t* sk = ring + stage * C::kStageBytes;
#pragma unroll
                    for (int hx = 0; hx < HD / 64; ++hx) {
                        ptx::tma_load_2d(sk + hx * C::kHalfBytes, &tm, &full[stage], hx * 64, rk + k0, pol);
                        ptx::tma_load_2d(sk + C::kChunkBytes + hx * C::kHalfBytes, &tm, &full[stage], hx * 64, rv + k0,
                                         pol);
                    }
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            ptx::mbar_wait(&q_empty[qs], qph ^ 1);  // end of work
            sq_item[qs] = -1;
            ptx::mbar_arrive(&q_full[qs]);
        }
        return;
    }

    // ---------------------------------------------------- compute warps 0-3
    // Chunk j of an item is processed entirely by warp j % 4 (64 keys = four
    // independent 16-key m-tiles).  The warps never synchronise with each
    // other: every warp steps through every ring position (waiting for the
    // chunk, using it if it is its own, releasing it -- the empty barrier
    // needs all four), keeps its own online softmax over its chunks of the
    // item, and publishes its (max, sum, O) as one contributor; the last of
    // the (sample, head, query tile)'s contributors folds them all in a fixed
    // order (split-major, warp-minor: deterministic).
    const int g = lane / 4, c = lane % 4;
    int pos = 0;  // ring position of the current item's first chunk
    int qs = 0;
    uint32_t qph = 0;
    for (;;) {
        ptx::mbar_wait(&q_full[qs], qph);  // the item's Q rows (or the end marker)
        const int i = sq_item[qs];
        if (i < 0) break;
        const Item it = item_at(a, i, splits, qtiles);
        const SampleSeg seg = a.segs[it.s];
        const int nchunks = (it.k_end - it.k_begin + kAttnChunk - 1) / kAttnChunk;
        uint32_t qf[HD / 32][4];  // Q^T B-fragments of every 32-wide hd slice, from the first stage's Q rows
        {
            const uint32_t qa = ptx::smem_u32(qring + qs * C::kQBytes);
#pragma unroll
            for (int kk = 0; kk < HD / 32; ++kk)
                ldsm_x4(qa + (lane % 8) * HD * 2 + (kk * 32 + (lane / 8) * 8) * 2, qf[kk][0], qf[kk][1], qf[kk][2],
                        qf[kk][3]);
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&q_empty[qs]);
            if (++qs == C::kQSlots) {
                qs = 0;
                qph ^= 1;
            }
        }
        // this lane's two query columns: token ids and causal limits (write slots)
        int tq[2], ws[2];
#pragma unroll
        for (int qi = 0; qi < 2; ++qi) {
            const int r = 2 * c + qi;
            tq[qi] = r < it.nq ? a.qidx[seg.q_start + it.qt * kAttnQT + r] : -1;
            ws[qi] = tq[qi] >= 0 ? a.plans[tq[qi]].write_slot : -1;
        }
        float m_run[2] = {-INFINITY, -INFINITY}, l_part[2] = {0.0f, 0.0f};
        float o[HD / 16][4];
#pragma unroll
        for (int n = 0; n < HD / 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.0f;

        for (int jc = warp; jc < nchunks; jc += 4) {  // this warp's chunks only
            const int stage = (pos + jc) % C::kStages;
            ptx::mbar_wait(&full[stage], (uint32_t)(((pos + jc) / C::kStages) & 1));
            if (!(a.dbg & 1)) {
                const int k0 = it.k_begin + jc * kAttnChunk;
                const uint32_t ka = ptx::smem_u32(ring + stage * C::kStageBytes);
                const uint32_t va = ka + C::kChunkBytes;
                // S^T = K Q^T : 64 keys (4 m-tiles) x 8 queries
                float st[4][4];
#pragma unroll
                for (int t = 0; t < 4; ++t) st[t][0] = st[t][1] = st[t][2] = st[t][3] = 0.0f;
#pragma unroll
                for (int kk = 0; kk < HD / 32; ++kk) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        uint32_t a0, a1, a2, a3, e0, e1, e2, e3;
                        ldsm_x4(ka + tswz(t * 16 + (lane % 16), kk * 32 + (lane / 16) * 8), a0, a1, a2, a3);
                        ldsm_x4(ka + tswz(t * 16 + (lane % 16), kk * 32 + 16 + (lane / 16) * 8), e0, e1, e2, e3);
                        mma_bf16(st[t], a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
                        mma_bf16(st[t], e0, e1, e2, e3, qf[kk][2], qf[kk][3]);
                    }
                }
                // mask (extent, causal write slot, padded-grid holes) and online softmax
                float cmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int key = k0 + t * 16 + g + (e >= 2 ? 8 : 0);
                        const int qi = e & 1;
                        const bool vis =
                            key < it.k_end && key <= ws[qi] && !(a.pad && a.pad[(size_t)it.s * a.cap + key]);
                        st[t][e] = vis ? st[t][e] * a.scale_log2 : -INFINITY;
                        cmax[qi] = fmaxf(cmax[qi], st[t][e]);
                    }
                }
                float alpha[2];
#pragma unroll
                for (int qi = 0; qi < 2; ++qi) {
                    cmax[qi] = fmaxf(cmax[qi], __shfl_xor_sync(0xffffffffu, cmax[qi], 4));
                    cmax[qi] = fmaxf(cmax[qi], __shfl_xor_sync(0xffffffffu, cmax[qi], 8));
                    cmax[qi] = fmaxf(cmax[qi], __shfl_xor_sync(0xffffffffu, cmax[qi], 16));
                    const float m_new = fmaxf(m_run[qi], cmax[qi]);
                    alpha[qi] = m_new == -INFINITY ? 1.0f : exp2f(m_run[qi] - m_new);  // exp2(-inf) = 0
                    m_run[qi] = m_new;
                }
                l_part[0] *= alpha[0];
                l_part[1] *= alpha[1];
#pragma unroll
                for (int n = 0; n < HD / 16; ++n) {
                    o[n][0] *= alpha[0];
                    o[n][2] *= alpha[0];
                    o[n][1] *= alpha[1];
                    o[n][3] *= alpha[1];
                }
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    float p[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        p[e] = m_run[e & 1] == -INFINITY ? 0.0f : exp2f(st[t][e] - m_run[e & 1]);
                    l_part[0] += p[0] + p[2];
                    l_part[1] += p[1] + p[3];
                    const uint32_t pb0 = movmatrix_t(pack_bf16(p[0], p[1]));  // keys 0-7 of m-tile t
                    const uint32_t pb1 = movmatrix_t(pack_bf16(p[2], p[3]));  // keys 8-15
                    // O^T += V^T P^T : per 16 hd rows (m-tile n), k = the 16 keys of m-tile t
#pragma unroll
                    for (int n = 0; n < HD / 16; ++n) {
                        uint32_t a0, a1, a2, a3;
                        ldsm_x4_t(va + tswz(t * 16 + (lane % 8) + ((lane / 16) * 8), n * 16 + ((lane / 8) % 2) * 8),
                                  a0, a1, a2, a3);
                        mma_bf16(o[n], a0, a1, a2, a3, pb0, pb1);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[stage]);
        }
        pos += nchunks;
        if (warp >= nchunks) continue;  // no chunk of this item: not a contributor

        // ------------------------------------------ publish this warp's contribution
#pragma unroll
        for (int qi = 0; qi < 2; ++qi) {
            l_part[qi] += __shfl_xor_sync(0xffffffffu, l_part[qi], 4);
            l_part[qi] += __shfl_xor_sync(0xffffffffu, l_part[qi], 8);
            l_part[qi] += __shfl_xor_sync(0xffffffffu, l_part[qi], 16);
        }
        // contributors of (sample, head, query tile): split-major, warp-minor
        int n_contrib = 0;
        for (int sp = 0; sp < it.nsplit; ++sp) {
            const int len = min(seg.kv_len, (sp + 1) * kAttnSplit) - sp * kAttnSplit;
            n_contrib += min(4, (len + kAttnChunk - 1) / kAttnChunk);
        }
        const int max_contrib = a.max_splits * 4;
        if (n_contrib == 1) {  // the whole extent was one chunk: write the context directly
#pragma unroll
            for (int qi = 0; qi < 2; ++qi) {
                if (tq[qi] < 0) continue;
                const float inv = 1.0f / l_part[qi];
#pragma unroll
                for (int n = 0; n < HD / 16; ++n) {
                    __nv_bfloat16* dst = a.ctx + (size_t)tq[qi] * a.h + it.head * HD + n * 16 + g;
                    dst[0] = __float2bfloat16_rn(o[n][qi] * inv);
                    dst[8] = __float2bfloat16_rn(o[n][qi + 2] * inv);
                }
            }
            continue;
        }
        const int slot = it.split * 4 + warp;
#pragma unroll
        for (int qi = 0; qi < 2; ++qi) {
            if (tq[qi] < 0) continue;
            const size_t b = ((size_t)tq[qi] * a.heads + it.head) * max_contrib + slot;
#pragma unroll
            for (int n = 0; n < HD / 16; ++n) {
                a.part_o[b * HD + n * 16 + g] = o[n][qi];
                a.part_o[b * HD + n * 16 + g + 8] = o[n][qi + 2];
            }
            if (g == 0) {
                a.part_ml[b * 2] = m_run[qi];
                a.part_ml[b * 2 + 1] = l_part[qi];
            }
        }
        __syncwarp();
        int last = 0;
        if (lane == 0) {
            // acq_rel RMW: this warp's partial (program-ordered before it, the
            // warp synchronised above) is released; the last arriver acquires all
            int* cnt = a.cnt + ((size_t)it.s * a.heads + it.head) * kMaxQTiles + it.qt;
            int old;
            asm volatile("fence.acq_rel.gpu;\n\tatom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
            last = old == n_contrib - 1;
            if (last) *cnt = 0;  // self-resetting for the next layer / graph replay
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) continue;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        // ------------------------------------------ fold every contributor (fixed order)
        for (int r = 0; r < it.nq; ++r) {
            const int tok = a.qidx[seg.q_start + it.qt * kAttnQT + r];
            const size_t b0 = ((size_t)tok * a.heads + it.head) * max_contrib;
            float M = -INFINITY;
            for (int sp = 0; sp < it.nsplit; ++sp) {
                const int len = min(seg.kv_len, (sp + 1) * kAttnSplit) - sp * kAttnSplit;
                const int nw = min(4, (len + kAttnChunk - 1) / kAttnChunk);
                for (int w = 0; w < nw; ++w) M = fmaxf(M, __ldcg(a.part_ml + (b0 + sp * 4 + w) * 2));
            }
            float L = 0.0f;
            float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int sp = 0; sp < it.nsplit; ++sp) {
                const int len = min(seg.kv_len, (sp + 1) * kAttnSplit) - sp * kAttnSplit;
                const int nw = min(4, (len + kAttnChunk - 1) / kAttnChunk);
                for (int w = 0; w < nw; ++w) {
                    const size_t b = b0 + sp * 4 + w;
                    const float mk = __ldcg(a.part_ml + b * 2);
                    if (mk == -INFINITY) continue;
                    const float f = exp2f(mk - M);
                    L += __ldcg(a.part_ml + b * 2 + 1) * f;
                    if (lane * 4 < HD) {
                        const float4 v = __ldcg((const float4*)(a.part_o + b * HD) + lane);
                        O.x += v.x * f;
                        O.y += v.y * f;
                        O.z += v.z * f;
                        O.w += v.w * f;
                    }
                }
            }
            if (lane * 4 < HD) {
                const float inv = 1.0f / L;
                __nv_bfloat162* dst = (__nv_bfloat162*)(a.ctx + (size_t)tok * a.h + it.head * HD + lane * 4);
                dst[0] = __floats2bfloat162_rn(O.x * inv, O.y * inv);
                dst[1] = __floats2bfloat162_rn(O.z * inv, O.w * inv);
            }
        }
    }
}

int g_sms = 148;

}  // namespace

CUtensorMap make_kv_map(const void* kv, int64_t rows, int hd) { return make_tmap_2d(kv, rows, hd, kAttnChunk); }

template <int HD, int S, int N>
void attn_attr() {
    CUDA_OK(cudaFuncSetAttribute(k_attention<HD, S, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<HD, S>::kSmem));
}

void attention_prepare() {
    static bool done = false;
    if (done) return;
    attn_attr<128, 6, 1>();
    attn_attr<64, 8, 1>();
    done = true;
}

template <int HD, int S, int N>
void attn_go(const AttnArgs& a, const CUtensorMap& kv_map, int splits, int qtiles, cudaStream_t st) {
    const int n_items = a.B * a.heads * qtiles * splits;
    const int grid = std::min(n_items, N * g_sms);
    launch_k(k_attention<HD, S, N>, dim3(grid), dim3(kThreads), ACfg<HD, S>::kSmem, st, kv_map, a, splits, qtiles);
}

void attention_launch(const AttnArgs& a, const CUtensorMap& kv_map, int hd, int splits, int qtiles, cudaStream_t st) {
    attention_prepare();
    SD_CHECK(qtiles <= kMaxQTiles, INTERNAL, "too many query tiles per sample");
    SD_CHECK(splits <= a.max_splits, INTERNAL, "too many KV splits");
    if (hd == 128)
        attn_go<128, 6, 1>(a, kv_map, splits, qtiles, st);  // 6 x 34 KB stages in flight per SM
    else if (hd == 64)
        attn_go<64, 8, 1>(a, kv_map, splits, qtiles, st);
    else
        throw Error(CONFIG, "bf16 mode supports head_dim 64 or 128");
    CUDA_OK(cudaGetLastError());
}

}  // namespace sdb
