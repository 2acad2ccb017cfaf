// Split-grid ragged attention (the default bf16 path): one CTA per (sample,
// head) x 128-key split x 8-query tile, 3 CTAs per SM, and a split-combine
// kernel.  attention_sm100.cu holds an experimental persistent TMA-ring
// variant (SD_ATTN_IMPL=2) that is not yet faster.
#include <cuda_bf16.h>

#include <algorithm>

#include "attn.h"
#include "pdl.cuh"
#include "trace.cuh"

SD_TRACE_TU(attn1)

namespace sdb {
namespace {
constexpr int kSplit = 128;
constexpr int kQT = 8;
// ------------------------------------------------------------- attention
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

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

// smem tile [rows][HD] bf16 with the 16-byte chunk index XOR-swizzled by row%8
template <int HD>
__device__ __forceinline__ uint32_t swz(int row, int col) {  // byte offset of element (row, col)
    constexpr int kChunks = HD / 8;
    int chunk = (col >> 3) ^ (row & 7);
    return (uint32_t)(row * kChunks + chunk) * 16 + (col & 7) * 2;
}



// Ragged multi-query attention, "keys as M" formulation.
//
// One CTA = (sample, head) x 128-key split x 8-query tile; 4 warps each own 32
// keys.  With only n_s <= 8 draft queries per sample, the tensor-core tile is
// transposed so the KEYS are the 16-row M side and the queries the 8-wide N
// side of mma.sync m16n8k16:  S^T = K Q^T  and  O^T += V^T P^T.  P^T is
// re-laid from the S^T accumulator fragments with movmatrix (no smem trip),
// the softmax reduces over keys with 3 shuffles, and the O^T accumulators are
// 32 registers per thread.  This halves the MMA count of a 16-query tile and
// keeps register pressure low enough for several CTAs per SM.  The 4 warps'
// (max, sum, O) states merge through smem; splits merge in k_attn_combine.
// A sample's K/V extent is read once per split, not once per query token (the
// paper's per-token grid, re-reads it n_s times).
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

template <int HD>
__global__ void __launch_bounds__(128) k_attention_v1(AttnArgs a) {
    CtaTrace trace__(TK_ATTN);
    pdl_trigger();
    pdl_wait();
    constexpr int kKeys = kSplit / 4;  // keys per warp (32)
    const int sh = blockIdx.x, split = blockIdx.y, qt = blockIdx.z;
    const int s = sh / a.heads, head = sh % a.heads;
    const SampleSeg seg = a.segs[s];
    const int k_begin = split * kSplit;
    if (seg.n_q == 0 || qt * kQT >= seg.n_q || k_begin >= seg.kv_len) return;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nq = min(kQT, seg.n_q - qt * kQT);

    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* sQ = sm;                                    // [8][HD]
    uint8_t* sK = sm + kQT * HD * 2 + warp * 2 * kKeys * HD * 2;
    uint8_t* sV = sK + kKeys * HD * 2;
    float* sMerge = (float*)(sm + kQT * HD * 2);         // reused: [4][8][HD] + [4][8][2]
    __shared__ int sWslot[kQT];
    __shared__ int sTok[kQT];

    const int kw0 = k_begin + warp * kKeys;
    const size_t kbase = ((((size_t)a.layer * 2 + 0) * a.B + s) * a.heads + head) * (size_t)a.cap * HD;
    const size_t vbase = ((((size_t)a.layer * 2 + 1) * a.B + s) * a.heads + head) * (size_t)a.cap * HD;
    const int kv_end = min(seg.kv_len, k_begin + kSplit);
    for (int i = lane; i < kKeys * HD / 8; i += 32) {  // this warp's K / V rows (zero past the extent)
        const int r = i / (HD / 8), c8 = i % (HD / 8);
        const int key = kw0 + r;
        const bool ok = key < kv_end;
        const size_t off = (size_t)(ok ? key : 0) * HD + c8 * 8;
        cp_async16(sK + swz<HD>(r, c8 * 8), a.kv + kbase + off, ok);
        cp_async16(sV + swz<HD>(r, c8 * 8), a.kv + vbase + off, ok);
    }
    for (int i = threadIdx.x; i < kQT * HD / 8; i += 128) {  // Q tile (rows >= nq zero)
        const int r = i / (HD / 8), c8 = i % (HD / 8);
        const int tok = r < nq ? a.qidx[seg.q_start + qt * kQT + r] : 0;
        cp_async16(sQ + swz<HD>(r, c8 * 8), a.q + (size_t)tok * a.h + head * HD + c8 * 8, r < nq);
    }
    if (threadIdx.x < kQT) {
        const int r = threadIdx.x;
        const int tok = r < nq ? a.qidx[seg.q_start + qt * kQT + r] : -1;
        sTok[r] = tok;
        sWslot[r] = tok >= 0 ? a.plans[tok].write_slot : -1;
    }
    cp_async_wait_all();
    __syncthreads();

    const int g = lane / 4, c = lane % 4;
    // running softmax state for this thread's two query columns q = 2c, 2c+1
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.0f, 0.0f};
    float o[HD / 16][4];  // O^T fragments: (hd d0+g / d0+g+8) x (q 2c, 2c+1)
#pragma unroll
    for (int n = 0; n < HD / 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.0f;

    if (kw0 < kv_end) {
        const uint32_t qa = (uint32_t)__cvta_generic_to_shared(sQ);
        const uint32_t ka = (uint32_t)__cvta_generic_to_shared(sK);
        const uint32_t va = (uint32_t)__cvta_generic_to_shared(sV);
        // S^T = K Q^T : (kKeys keys) x (8 queries), as kKeys/16 m-tiles
        float st[kKeys / 16][4];
#pragma unroll
        for (int t = 0; t < kKeys / 16; ++t) st[t][0] = st[t][1] = st[t][2] = st[t][3] = 0.0f;
#pragma unroll
        for (int kk = 0; kk < HD; kk += 32) {
            // B = Q^T for two k-steps: matrices (q 0-7, hd kk), (kk+8), (kk+16), (kk+24)
            uint32_t b0, b1, b2, b3;
            ldsm_x4(qa + swz<HD>(lane % 8, kk + (lane / 8) * 8), b0, b1, b2, b3);
#pragma unroll
            for (int t = 0; t < kKeys / 16; ++t) {
                uint32_t a0, a1, a2, a3, e0, e1, e2, e3;
                // A = K rows t*16.. : (keys 0-7, kk), (keys 8-15, kk), (keys 0-7, kk+8), (keys 8-15, kk+8)
                ldsm_x4(ka + swz<HD>(t * 16 + (lane % 16), kk + (lane / 16) * 8), a0, a1, a2, a3);
                ldsm_x4(ka + swz<HD>(t * 16 + (lane % 16), kk + 16 + (lane / 16) * 8), e0, e1, e2, e3);
                mma_bf16(st[t], a0, a1, a2, a3, b0, b1);
                mma_bf16(st[t], e0, e1, e2, e3, b2, b3);
            }
        }
        // mask + max over this warp's keys for each query column
        const int ws[2] = {sWslot[2 * c], sWslot[2 * c + 1]};
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int t = 0; t < kKeys / 16; ++t) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = kw0 + t * 16 + g + (e >= 2 ? 8 : 0);
                const int qi = e & 1;
                const bool vis = key < kv_end && key <= ws[qi] && !(a.pad && a.pad[(size_t)s * a.cap + key]);
                const float x = vis ? st[t][e] * a.scale_log2 : -INFINITY;
                st[t][e] = x;
                mx[qi] = fmaxf(mx[qi], x);
            }
        }
#pragma unroll
        for (int qi = 0; qi < 2; ++qi) {
            mx[qi] = fmaxf(mx[qi], __shfl_xor_sync(0xffffffffu, mx[qi], 4));
            mx[qi] = fmaxf(mx[qi], __shfl_xor_sync(0xffffffffu, mx[qi], 8));
            mx[qi] = fmaxf(mx[qi], __shfl_xor_sync(0xffffffffu, mx[qi], 16));
            m_run[qi] = mx[qi];
        }
        float sum[2] = {0.0f, 0.0f};
        uint32_t pb[kKeys / 16][2];  // P^T as mma B fragments (keys 2c.. / 2c+8.., q g)
#pragma unroll
        for (int t = 0; t < kKeys / 16; ++t) {
            const float p0 = m_run[0] == -INFINITY ? 0.0f : exp2f(st[t][0] - m_run[0]);
            const float p1 = m_run[1] == -INFINITY ? 0.0f : exp2f(st[t][1] - m_run[1]);
            const float p2 = m_run[0] == -INFINITY ? 0.0f : exp2f(st[t][2] - m_run[0]);
            const float p3 = m_run[1] == -INFINITY ? 0.0f : exp2f(st[t][3] - m_run[1]);
            sum[0] += p0 + p2;
            sum[1] += p1 + p3;
            pb[t][0] = movmatrix_t(pack_bf16(p0, p1));  // rows = keys 0-7 of the tile
            pb[t][1] = movmatrix_t(pack_bf16(p2, p3));  // rows = keys 8-15
        }
#pragma unroll
        for (int qi = 0; qi < 2; ++qi) {
            sum[qi] += __shfl_xor_sync(0xffffffffu, sum[qi], 4);
            sum[qi] += __shfl_xor_sync(0xffffffffu, sum[qi], 8);
            sum[qi] += __shfl_xor_sync(0xffffffffu, sum[qi], 16);
            l_run[qi] = sum[qi];
        }
        // O^T += V^T P^T : per 16 keys (k-step) and 16 hd rows (m-tile)
#pragma unroll
        for (int t = 0; t < kKeys / 16; ++t) {
#pragma unroll
            for (int n = 0; n < HD / 16; ++n) {
                uint32_t a0, a1, a2, a3;
                // A = V^T (hd x keys): trans of V blocks (keys t*16+[0,8)/[8,16), hd n*16+[0,8)/[8,16))
                const int key = t * 16 + (lane % 8) + ((lane / 16) * 8);
                const int col = n * 16 + ((lane / 8) % 2) * 8;
                ldsm_x4_t(va + swz<HD>(key, col), a0, a1, a2, a3);
                mma_bf16(o[n], a0, a1, a2, a3, pb[t][0], pb[t][1]);
            }
        }
    }
    __syncthreads();  // every warp is done with K / V: reuse the area for the merge
    float* mO = sMerge + (size_t)warp * kQT * HD;   // [q][hd]
    float* mML = sMerge + 4 * kQT * HD + warp * 2 * kQT;
#pragma unroll
    for (int n = 0; n < HD / 16; ++n) {
        mO[(2 * c) * HD + n * 16 + g] = o[n][0];
        mO[(2 * c + 1) * HD + n * 16 + g] = o[n][1];
        mO[(2 * c) * HD + n * 16 + g + 8] = o[n][2];
        mO[(2 * c + 1) * HD + n * 16 + g + 8] = o[n][3];
    }
    if (g == 0) {
        mML[(2 * c) * 2] = m_run[0];
        mML[(2 * c) * 2 + 1] = l_run[0];
        mML[(2 * c + 1) * 2] = m_run[1];
        mML[(2 * c + 1) * 2 + 1] = l_run[1];
    }
    __syncthreads();
    const int nsplit = (seg.kv_len + kSplit - 1) / kSplit;
    for (int i = threadIdx.x; i < kQT * HD; i += 128) {
        const int r = i / HD, d = i % HD;
        if (r >= nq) continue;
        float M = -INFINITY;
        for (int w = 0; w < 4; ++w) M = fmaxf(M, sMerge[4 * kQT * HD + w * 2 * kQT + r * 2]);
        float L = 0.0f, O = 0.0f;
        for (int w = 0; w < 4; ++w) {
            const float mw = sMerge[4 * kQT * HD + w * 2 * kQT + r * 2];
            if (mw == -INFINITY) continue;
            const float f = exp2f(mw - M);
            L += sMerge[4 * kQT * HD + w * 2 * kQT + r * 2 + 1] * f;
            O += sMerge[(size_t)w * kQT * HD + r * HD + d] * f;
        }
        const int tok = sTok[r];
        if (nsplit == 1) {
            a.ctx[(size_t)tok * a.h + head * HD + d] = __float2bfloat16_rn(O / L);
        } else {
            const size_t base = ((size_t)tok * a.heads + head) * a.max_splits + split;
            a.part_o[base * HD + d] = O;
            if (d == 0) {
                a.part_ml[base * 2] = M;
                a.part_ml[base * 2 + 1] = L;
            }
        }
    }
}

// merge split-KV partials: grid (T, heads), block HD
__global__ void k_attn_combine_v1(AttnArgs a, int hd, const int* __restrict__ dT) {
    CtaTrace trace__(TK_ATTN_COMBINE);
    pdl_trigger();
    pdl_wait();
    int t = blockIdx.x, head = blockIdx.y, d = threadIdx.x;
    if (t >= *dT) return;
    int s = a.plans[t].sample;
    int nsplit = (a.segs[s].kv_len + kSplit - 1) / kSplit;
    if (nsplit <= 1) return;
    size_t base = ((size_t)t * a.heads + head) * a.max_splits;
    float M = -INFINITY;
    for (int k = 0; k < nsplit; ++k) M = fmaxf(M, a.part_ml[(base + k) * 2]);
    float L = 0.0f, O = 0.0f;
    for (int k = 0; k < nsplit; ++k) {
        float mk = a.part_ml[(base + k) * 2];
        if (mk == -INFINITY) continue;
        float f = exp2f(mk - M);
        L += a.part_ml[(base + k) * 2 + 1] * f;
        O += a.part_o[(base + k) * hd + d] * f;
    }
    a.ctx[(size_t)t * a.h + head * hd + d] = __float2bfloat16_rn(O / L);
}

}  // namespace

void attention_v1_launch(const AttnArgs& a, int hd, int max_kv_upper, int max_q_upper, int T_upper, const int* dT,
                         cudaStream_t st) {
    static bool prepared = false;
    if (!prepared) {
        CUDA_OK(cudaFuncSetAttribute(k_attention_v1<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_OK(cudaFuncSetAttribute(k_attention_v1<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        prepared = true;
    }
    const int splits = std::max(1, (max_kv_upper + kSplit - 1) / kSplit);
    const int qtiles = std::max(1, (max_q_upper + kQT - 1) / kQT);
    AttnArgs b = a;
    b.max_splits = a.max_splits * 4;  // the partial buffers hold 4 contributors per 512-key split
    SD_CHECK(splits <= b.max_splits, INTERNAL, "attention: too many splits for the partial buffers");
    const size_t smem = (size_t)kQT * hd * 2 + (size_t)4 * 2 * (kSplit / 4) * hd * 2;
    if (hd == 128)
        launch_k(k_attention_v1<128>, dim3(a.B * a.heads, splits, qtiles), dim3(128), smem, st, b);
    else
        launch_k(k_attention_v1<64>, dim3(a.B * a.heads, splits, qtiles), dim3(128), smem, st, b);
    if (splits > 1) launch_k(k_attn_combine_v1, dim3(T_upper, a.heads), dim3(hd), 0, st, b, hd, dT);
    CUDA_OK(cudaGetLastError());
}

}  // namespace sdb
