// fp32 CHECK mode: the verify-step forward with the reference's exact
// arithmetic, for bit-exact parity with the CPU
// oracle.  Every float operation is an explicitly rounded intrinsic
// (__fadd_rn / __fmul_rn / __fdiv_rn) so nvcc cannot contract to FFMA, every
// reduction runs in the reference's ascending order, and expf / tanhf are the
// glibc-faithful ports in glibc_mathf.h.  This mode is for correctness, not
// speed; the bf16 performance path lives in fast_kernels.cu / gemm_sm100.cu.
#include "common.h"
#include "glibc_mathf.h"

namespace sdb {
namespace {

// model.cpp:287-294: h = tok_emb[id] + pos_emb[logical_pos]
__global__ void k_embed(const float* __restrict__ w, int64_t tok_off, int64_t pos_off, int h,
                        const int32_t* __restrict__ tokens, const Plan* __restrict__ plans,
                        float* __restrict__ resid) {
    int t = blockIdx.x;
    const float* e = w + tok_off + (int64_t)tokens[t] * h;
    const float* p = w + pos_off + (int64_t)plans[t].logical_pos * h;
    for (int i = threadIdx.x; i < h; i += blockDim.x)
        resid[(int64_t)t * h + i] = __fadd_rn(e[i], p[i]);
}

// model.cpp:57-69, one block per row.  Mean / variance are serial by thread 0
// (the reference's single-accumulator ascending loops).
__global__ void k_layernorm(const float* __restrict__ x, const float* __restrict__ g,
                            const float* __restrict__ b, int dim, float* __restrict__ y) {
    __shared__ float s_mean, s_inv;
    const float* row = x + (int64_t)blockIdx.x * dim;
    if (threadIdx.x == 0) {
        float mean = 0.0f;
        for (int i = 0; i < dim; ++i) mean = __fadd_rn(mean, row[i]);
        mean = __fdiv_rn(mean, (float)dim);
        float var = 0.0f;
        for (int i = 0; i < dim; ++i) {
            float d = __fsub_rn(row[i], mean);
            var = __fadd_rn(var, __fmul_rn(d, d));
        }
        var = __fdiv_rn(var, (float)dim);
        s_mean = mean;
        s_inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
    }
    __syncthreads();
    float mean = s_mean, inv = s_inv;
    float* out = y + (int64_t)blockIdx.x * dim;
    for (int i = threadIdx.x; i < dim; i += blockDim.x)
        out[i] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(row[i], mean), inv), g[i]), b[i]);
}

// model.cpp:47-55: y[t][o] = b[o] + sum_i W[o][i] * x[t][i], ascending i,
// accumulator seeded with the bias (or 0 for the LM head).  Each thread owns
// one output feature for a tile of kTok tokens so every weight is read once
// per tile; each (t, o) chain is still the reference's serial order.
constexpr int kTok = 8;
__global__ void k_linear(const float* __restrict__ W, const float* __restrict__ bias, int out_dim,
                         int in_dim, const float* __restrict__ X, int ldx, float* __restrict__ Y,
                         int ldy, int T) {
    int o = blockIdx.x * blockDim.x + threadIdx.x;
    int t0 = blockIdx.y * kTok;
    int nt = min(kTok, T - t0);
    extern __shared__ float xs[];  // [kTok][chunk]
    const int chunk = 256;
    float acc[kTok];
    float b0 = (bias != nullptr && o < out_dim) ? bias[o] : 0.0f;
#pragma unroll
    for (int j = 0; j < kTok; ++j) acc[j] = b0;
    const float* wrow = W + (int64_t)(o < out_dim ? o : 0) * in_dim;
    for (int c0 = 0; c0 < in_dim; c0 += chunk) {
        int cn = min(chunk, in_dim - c0);
        __syncthreads();
        for (int idx = threadIdx.x; idx < kTok * chunk; idx += blockDim.x) {
            int j = idx / chunk, i = idx % chunk;
            xs[idx] = (j < nt && i < cn) ? X[(int64_t)(t0 + j) * ldx + c0 + i] : 0.0f;
        }
        __syncthreads();
        if (o < out_dim) {
            for (int i = 0; i < cn; ++i) {
                float w = wrow[c0 + i];
#pragma unroll
                for (int j = 0; j < kTok; ++j) acc[j] = __fadd_rn(acc[j], __fmul_rn(w, xs[j * chunk + i]));
            }
        }
    }
    if (o < out_dim)
        for (int j = 0; j < nt; ++j) Y[(int64_t)(t0 + j) * ldy + o] = acc[j];
}

// UnpadArena::write_kv / PaddedGrid::write_kv (kv_cache.cpp:128-138, 203-213)
// for every token with store=1; qkv rows are [q | k | v].
__global__ void k_kv_write(const float* __restrict__ qkv, const Plan* __restrict__ plans, int h,
                           int heads, int hd, int B, int cap, int layer, float* __restrict__ kv) {
    int t = blockIdx.x;
    Plan p = plans[t];
    if (!p.store) return;
    for (int i = threadIdx.x; i < h; i += blockDim.x) {
        int head = i / hd, d = i % hd;
        size_t ko = ((((size_t)layer * 2 + 0) * B + p.sample) * heads + head) * (size_t)cap * hd +
                    (size_t)p.write_slot * hd + d;
        size_t vo = ((((size_t)layer * 2 + 1) * B + p.sample) * heads + head) * (size_t)cap * hd +
                    (size_t)p.write_slot * hd + d;
        kv[ko] = qkv[(int64_t)t * 3 * h + h + i];
        kv[vo] = qkv[(int64_t)t * 3 * h + 2 * h + i];
    }
}

// model.cpp:320-349 + gather_visible (kv_cache.cpp:140-150, 221-235): one block
// per (token, head).  Visible rows are slots [0, write_slot] of the token's own
// sample, skipping pad rows of the padded grid, in ascending order.
__global__ void k_attention(const float* __restrict__ qkv, const Plan* __restrict__ plans,
                            const float* __restrict__ kv, const uint8_t* __restrict__ pad, int h,
                            int heads, int hd, int B, int cap, int layer, float scale,
                            float* __restrict__ scores_ws, int32_t* __restrict__ rows_ws,
                            float* __restrict__ ctx, int32_t* __restrict__ err) {
    int t = blockIdx.x, head = blockIdx.y;
    Plan p = plans[t];
    float* scores = scores_ws + ((size_t)t * heads + head) * cap;
    int32_t* rows = rows_ws + ((size_t)t * heads + head) * cap;
    __shared__ int s_count;
    __shared__ float s_max, s_denom;
    if (threadIdx.x == 0) {
        int n = 0;
        for (int r = 0; r <= p.write_slot; ++r) {
            if (pad != nullptr && pad[(size_t)p.sample * cap + r]) continue;
            rows[n++] = r;
        }
        s_count = n;
        if (n < 1) atomicExch(err, 3);  // "token with an empty visible set"
    }
    __syncthreads();
    int count = s_count;
    if (count < 1) return;
    const float* q = qkv + (int64_t)t * 3 * h + head * hd;
    const float* kbase = kv + ((((size_t)layer * 2 + 0) * B + p.sample) * heads + head) * (size_t)cap * hd;
    const float* vbase = kv + ((((size_t)layer * 2 + 1) * B + p.sample) * heads + head) * (size_t)cap * hd;
    for (int j = threadIdx.x; j < count; j += blockDim.x) {
        const float* k = kbase + (size_t)rows[j] * hd;
        float acc = 0.0f;
        for (int d = 0; d < hd; ++d) acc = __fadd_rn(acc, __fmul_rn(q[d], k[d]));
        scores[j] = __fmul_rn(acc, scale);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float mx = scores[0];
        for (int j = 1; j < count; ++j) mx = (mx < scores[j]) ? scores[j] : mx;  // std::max
        s_max = mx;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < count; j += blockDim.x) scores[j] = sd_expf(__fsub_rn(scores[j], s_max));
    __syncthreads();
    if (threadIdx.x == 0) {
        float den = 0.0f;
        for (int j = 0; j < count; ++j) den = __fadd_rn(den, scores[j]);
        s_denom = den;
    }
    __syncthreads();
    float den = s_denom;
    for (int d = threadIdx.x; d < hd; d += blockDim.x) {
        float c = 0.0f;
        for (int j = 0; j < count; ++j) {
            float wgt = __fdiv_rn(scores[j], den);
            c = __fadd_rn(c, __fmul_rn(wgt, vbase[(size_t)rows[j] * hd + d]));
        }
        ctx[(int64_t)t * h + head * hd + d] = c;
    }
}

__global__ void k_residual_add(float* __restrict__ resid, const float* __restrict__ delta, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        resid[i] = __fadd_rn(resid[i], delta[i]);
}

// model.cpp:71-74
__global__ void k_gelu(float* __restrict__ x, int64_t n) {
    const float c = 0.7978845608028654f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float v = x[i];
        float cube = __fmul_rn(__fmul_rn(__fmul_rn(0.044715f, v), v), v);
        float th = sd_tanhf(__fmul_rn(c, __fadd_rn(v, cube)));
        x[i] = __fmul_rn(__fmul_rn(0.5f, v), __fadd_rn(1.0f, th));
    }
}

}  // namespace

// model.cpp:34-41 greedy_next (strict >, lowest id on ties) + the isfinite
// check of model.cpp:368-370.  One block per row.
__global__ void k_row_argmax(const float* __restrict__ logits, int V, int32_t* __restrict__ out,
                             int32_t* __restrict__ nonfinite) {
    const float* row = logits + (int64_t)blockIdx.x * V;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    bool bad = false;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        float v = row[i];
        if (!isfinite(v)) bad = true;
        if (bi == 0x7fffffff || v > bv) {
            bv = v;
            bi = i;
        }
    }
    __shared__ float sv[32];
    __shared__ int si[32];
    for (int off = 16; off > 0; off >>= 1) {
        float ov = __shfl_down_sync(0xffffffff, bv, off);
        int oi = __shfl_down_sync(0xffffffff, bi, off);
        if (oi != 0x7fffffff && (bi == 0x7fffffff || ov > bv || (ov == bv && oi < bi))) {
            bv = ov;
            bi = oi;
        }
    }
    if (bad) atomicExch(nonfinite, 1);
    int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
    if (lane == 0) {
        sv[wid] = bv;
        si[wid] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x / 32); ++w) {
            if (si[w] != 0x7fffffff && (si[0] == 0x7fffffff || sv[w] > sv[0] || (sv[w] == sv[0] && si[w] < si[0]))) {
                sv[0] = sv[w];
                si[0] = si[w];
            }
        }
        out[blockIdx.x] = si[0];
    }
}

static int blocks_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)(g < 148 * 8 ? (g < 1 ? 1 : g) : 148 * 8);
}

static void linear(const float* W, const float* b, int out_dim, int in_dim, const float* X, int ldx,
                   float* Y, int ldy, int T, cudaStream_t st) {
    dim3 grid((out_dim + 127) / 128, (T + kTok - 1) / kTok);
    k_linear<<<grid, 128, sizeof(float) * kTok * 256, st>>>(W, b, out_dim, in_dim, X, ldx, Y, ldy, T);
}

void forward_check(const Model& m, Cache& c, Workspace& ws, int T, bool /*want_logits*/,
                   cudaStream_t st) {
    const Config& cfg = m.cfg;
    const WeightLayout& L = m.lay;
    int h = cfg.hidden(), mm = cfg.mlp(), heads = cfg.num_heads, hd = cfg.head_dim, V = cfg.vocab_size;
    float scale = 1.0f / sqrtf((float)hd);  // model.cpp:271 (host, correctly rounded)
    const float* W = m.w32;
    float* kv = (float*)c.kv;
    float* resid = ws.d_resid;
    float* xln = ws.d_tmp;                 // [T, h]
    float* qkv = ws.d_tmp2;                // [T, 3h]
    float* ctx = ws.d_tmp + (size_t)T * h; // [T, h]
    float* mlp = ws.d_tmp2 + (size_t)T * 3 * h;  // [T, m]
    float* outb = ws.d_tmp + (size_t)2 * T * h;  // [T, h]
    int32_t* rows_ws = (int32_t*)(ws.d_scores + (size_t)T * heads * c.cap);
    const uint8_t* pad = c.layout == PADDED ? c.d_pad : nullptr;

    k_embed<<<T, 128, 0, st>>>(W, L.tok, L.pos, h, ws.d_tokens, ws.d_plans, resid);
    for (int l = 0; l < cfg.num_layers; ++l) {
        const LayerOff& o = L.layer[l];
        // phase 1 (model.cpp:307-318): LN1, Q/K/V, cache writes for all tokens
        k_layernorm<<<T, 128, 0, st>>>(resid, W + o.ln1_g, W + o.ln1_b, h, xln);
        linear(W + o.wq, W + o.bq, h, h, xln, h, qkv, 3 * h, T, st);
        linear(W + o.wk, W + o.bk, h, h, xln, h, qkv + h, 3 * h, T, st);
        linear(W + o.wv, W + o.bv, h, h, xln, h, qkv + 2 * h, 3 * h, T, st);
        k_kv_write<<<T, 128, 0, st>>>(qkv, ws.d_plans, h, heads, hd, c.B, c.cap, l, kv);
        // phase 2 (model.cpp:320-358)
        k_attention<<<dim3(T, heads), 128, 0, st>>>(qkv, ws.d_plans, kv, pad, h, heads, hd, c.B, c.cap,
                                                    l, scale, ws.d_scores, rows_ws, ctx, ws.d_flag);
        linear(W + o.wo, W + o.bo, h, h, ctx, h, outb, h, T, st);
        k_residual_add<<<blocks_for((int64_t)T * h), 256, 0, st>>>(resid, outb, (int64_t)T * h);
        k_layernorm<<<T, 128, 0, st>>>(resid, W + o.ln2_g, W + o.ln2_b, h, xln);
        linear(W + o.w_fc, W + o.b_fc, mm, h, xln, h, mlp, mm, T, st);
        k_gelu<<<blocks_for((int64_t)T * mm), 256, 0, st>>>(mlp, (int64_t)T * mm);
        linear(W + o.w_proj, W + o.b_proj, h, mm, mlp, mm, outb, h, T, st);
        k_residual_add<<<blocks_for((int64_t)T * h), 256, 0, st>>>(resid, outb, (int64_t)T * h);
    }
    // model.cpp:361-371
    k_layernorm<<<T, 128, 0, st>>>(resid, W + L.lnf_g, W + L.lnf_b, h, xln);
    linear(W + L.lm, nullptr, V, h, xln, h, ws.d_logits, V, T, st);
    k_row_argmax<<<T, 256, 0, st>>>(ws.d_logits, V, ws.d_argmax, ws.d_flag);
    CUDA_OK(cudaGetLastError());
}

}  // namespace sdb
