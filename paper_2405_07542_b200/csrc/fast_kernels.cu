// bf16 PERFORMANCE mode forward of the verify step.
//
// Per layer (model.cpp:303-359, restructured for the GPU):
//   LN1 (fp32 residual -> bf16)          k_layernorm
//   QKV  tcgen05 GEMM + scatter epilogue  Q -> q16, K/V -> unpadded arena
//   ragged multi-query attention          attention_sm100.cu (persistent, in-kernel split combine)
//   O    tcgen05 GEMM + residual epilogue
//   LN2                                   k_layernorm
//   FC   tcgen05 GEMM + GELU epilogue
//   PROJ tcgen05 GEMM + residual epilogue
// then final LN, LM-head GEMM with the (max, lowest id) argmax epilogue, and
// k_argmax_reduce over the vocab tiles.  Weights and KV are bf16; the
// residual stream, accumulators and softmax are fp32.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "attn.h"
#include "gemm.h"
#include "handles.h"
#include "pdl.cuh"
#include "trace.cuh"

SD_TRACE_TU(fast)

namespace sdb {

constexpr int kChunkTokens = 256;  // tokens per forward chunk (GEMM N <= 256)
constexpr int kSms = 148;          // B200 SM count (stream-K GEMM grid)

struct FastModelState {
    std::vector<GemmMaps> qkv, o, fc, proj;  // per layer (A map only used)
    GemmMaps lm;
};

struct FastWorkspace {
    int cap_tokens = 0, B = 0, cap = 0, max_splits = 0;
    __nv_bfloat16 *xb = nullptr, *q = nullptr, *ctx = nullptr, *act = nullptr;
    float* part_o = nullptr;   // [T][heads][max_splits][hd]
    float* part_ml = nullptr;  // [T][heads][max_splits][2]
    float* part[2] = {nullptr, nullptr};  // stream-K partial sums, alternating between chained GEMMs
    int* gemm_cnt = nullptr;   // per GEMM call site: kGemmCntInts counters, zeroed per forward
    int n_sites = 0;
    float* arg_v = nullptr;    // LM-head per-tile argmax partials [256][kGemmMaxTiles]
    int* arg_i = nullptr;
    int* attn_cnt = nullptr;   // split-KV arrival counters [B * heads * kMaxQTiles]
    CUtensorMap kv_map;        // TMA view of the cache's KV arena
    GemmMaps map_xb, map_ctx, map_act;
    // per GEMM call site: the model's weight map + this workspace's token maps
    std::vector<GemmMaps> map_qkv, map_o, map_fc, map_proj;
    GemmMaps map_lm;
    std::vector<void*> allocs;
};

void free_fast_model(FastModelState* f) { delete f; }
void free_fast_workspace(FastWorkspace* f) {
    if (!f) return;
    for (void* p : f->allocs) dfree(p);
    delete f;
}

void build_fast_model(Model& m) {
    const Config& c = m.cfg;
    int64_t h = c.hidden(), mm = c.mlp();
    SD_CHECK(h % 64 == 0, CONFIG, "bf16 mode needs hidden % 64 == 0");
    SD_CHECK(c.head_dim == 64 || c.head_dim == 128, CONFIG, "bf16 mode supports head_dim 64 or 128");
    SD_CHECK(c.num_layers <= 256, CONFIG, "bf16 mode supports up to 256 layers");
    auto* f = new FastModelState();
    for (const FastLayer& L : m.layers) {
        GemmMaps g;
        g.A = make_tmap_2d(L.wqkv, 3 * h, h, kGemmTile);
        f->qkv.push_back(g);
        g.A = make_tmap_2d(L.wo, h, h, kGemmTile);
        f->o.push_back(g);
        g.A = make_tmap_2d(L.wfc, mm, h, kGemmTile);
        f->fc.push_back(g);
        g.A = make_tmap_2d(L.wproj, h, mm, kGemmTile);
        f->proj.push_back(g);
    }
    f->lm.A = make_tmap_2d(m.lm16, m.vocab_pad, h, kGemmTile);
    m.fast = f;
}

namespace {

// ------------------------------------------------------------- row kernels
template <typename F>
__device__ __forceinline__ float block_sum(float v, F* scratch) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    int w = threadIdx.x / 32, l = threadIdx.x % 32;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    float t = 0.0f;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) t += scratch[i];
    return t;
}

constexpr int kRowThreads = 256, kMaxPerThread = 32;  // hidden <= 8192

// LayerNorm of fp32 rows into bf16 (two-pass mean / variance, eps 1e-5).
__device__ __forceinline__ void ln_row(const float* x, const float* g, const float* b, int h,
                                       __nv_bfloat16* y, float* scratch) {
    float v[kMaxPerThread];
    int n = 0;
    float s = 0.0f;
    for (int i = threadIdx.x; i < h; i += kRowThreads) s += (v[n++] = x[i]);
    float mean = block_sum(s, scratch) / h;
    float q = 0.0f;
    for (int k = 0; k < n; ++k) {
        float d = v[k] - mean;
        q += d * d;
    }
    float inv = rsqrtf(block_sum(q, scratch) / h + 1e-5f);
    n = 0;
    for (int i = threadIdx.x; i < h; i += kRowThreads, ++n) y[i] = __float2bfloat16_rn((v[n] - mean) * inv * g[i] + b[i]);
}

__global__ void __launch_bounds__(kRowThreads) k_layernorm(const float* __restrict__ x, const float* __restrict__ g,
                                                           const float* __restrict__ b, int h,
                                                           __nv_bfloat16* __restrict__ y, const int* __restrict__ dT) {
    __shared__ float scratch[32];
    int t = blockIdx.x;
    if (t >= *dT) return;
    ln_row(x + (size_t)t * h, g, b, h, y + (size_t)t * h, scratch);
}

// embedding (model.cpp:287-294) fused with layer 0's LN1
__global__ void __launch_bounds__(kRowThreads) k_embed_ln(const __nv_bfloat16* __restrict__ tok,
                                                          const __nv_bfloat16* __restrict__ pos,
                                                          const int32_t* __restrict__ tokens,
                                                          const Plan* __restrict__ plans, int h,
                                                          float* __restrict__ resid, const float* __restrict__ g,
                                                          const float* __restrict__ b, __nv_bfloat16* __restrict__ y,
                                                          const int* __restrict__ dT) {
    CtaTrace trace__(TK_EMBED_LN);
    pdl_trigger();
    pdl_wait();
    __shared__ float scratch[32];
    int t = blockIdx.x;
    if (t >= *dT) return;
    const __nv_bfloat16* e = tok + (size_t)tokens[t] * h;
    const __nv_bfloat16* p = pos + (size_t)plans[t].logical_pos * h;
    float* r = resid + (size_t)t * h;
    for (int i = threadIdx.x; i < h; i += kRowThreads) r[i] = __bfloat162float(e[i]) + __bfloat162float(p[i]);
    __syncthreads();
    ln_row(r, g, b, h, y + (size_t)t * h, scratch);
}

// per-token argmax over the LM-head tile partials (lowest id on ties)
__global__ void k_argmax_reduce(const float* __restrict__ pv, const int* __restrict__ pi, int m_tiles, int ld,
                                int32_t* __restrict__ out, const int* __restrict__ dT) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= *dT) return;
    float bv = pv[t];
    int bi = pi[t];
    for (int k = 1; k < m_tiles; ++k) {
        float v = pv[(size_t)k * ld + t];
        int i = pi[(size_t)k * ld + t];
        if (v > bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
        }
    }
    out[t] = bi;
}

template <typename T>
T* walloc(FastWorkspace* f, size_t n) {
    T* p = (T*)dmalloc(sizeof(T) * (n ? n : 1));
    f->allocs.push_back(p);
    return p;
}

FastWorkspace* ensure_fast(const Model& m, const Cache& c, Workspace& ws) {
    FastWorkspace* f = ws.fast;
    int max_splits = (c.cap + kAttnSplit - 1) / kAttnSplit;
    if (f && f->B >= c.B && f->cap >= c.cap && f->max_splits >= max_splits) return f;
    free_fast_workspace(f);
    f = new FastWorkspace();
    const Config& cfg = m.cfg;
    size_t h = cfg.hidden(), mm = cfg.mlp(), T = kChunkTokens;
    f->cap_tokens = (int)T;
    f->B = c.B;
    f->cap = c.cap;
    f->max_splits = max_splits;
    f->xb = walloc<__nv_bfloat16>(f, T * h);
    f->q = walloc<__nv_bfloat16>(f, T * h);
    f->ctx = walloc<__nv_bfloat16>(f, T * h);
    f->act = walloc<__nv_bfloat16>(f, T * mm);
    f->part_o = walloc<float>(f, T * cfg.num_heads * max_splits * 4 * cfg.head_dim);  // 4 warp contributors per split
    f->part_ml = walloc<float>(f, T * cfg.num_heads * max_splits * 4 * 2);
    size_t part = 0;
    for (auto mk : {std::make_pair((int)(3 * h), (int)h), std::make_pair((int)h, (int)h),
                    std::make_pair((int)mm, (int)h), std::make_pair((int)h, (int)mm),
                    std::make_pair(m.vocab_pad, (int)h)})
        part = std::max(part, gemm_part_floats(mk.first, mk.second, kSms));
    f->part[0] = walloc<float>(f, part);
    f->part[1] = walloc<float>(f, part);
    f->n_sites = cfg.num_layers * 4 + 1;
    f->gemm_cnt = walloc<int>(f, (size_t)f->n_sites * kGemmCntInts + 256);  // + attention item counters
    f->arg_v = walloc<float>(f, (size_t)256 * kGemmMaxTiles);
    f->arg_i = walloc<int>(f, (size_t)256 * kGemmMaxTiles);
    f->attn_cnt = walloc<int>(f, (size_t)c.B * cfg.num_heads * kMaxQTiles);
    CUDA_OK(cudaMemset(f->attn_cnt, 0, sizeof(int) * (size_t)c.B * cfg.num_heads * kMaxQTiles));
    f->kv_map = make_kv_map(c.kv, (int64_t)cfg.num_layers * 2 * c.B * cfg.num_heads * c.cap, cfg.head_dim);
    make_b_maps(f->map_xb, f->xb, T, h);
    make_b_maps(f->map_ctx, f->ctx, T, h);
    make_b_maps(f->map_act, f->act, T, mm);
    const FastModelState* fm = m.fast;
    for (int l = 0; l < cfg.num_layers; ++l) {
        GemmMaps g = f->map_xb;
        g.A = fm->qkv[l].A;
        f->map_qkv.push_back(g);
        g = f->map_ctx;
        g.A = fm->o[l].A;
        f->map_o.push_back(g);
        g = f->map_xb;
        g.A = fm->fc[l].A;
        f->map_fc.push_back(g);
        g = f->map_act;
        g.A = fm->proj[l].A;
        f->map_proj.push_back(g);
    }
    f->map_lm = f->map_xb;
    f->map_lm.A = fm->lm.A;
    ws.fast = f;
    return f;
}

}  // namespace

// ------------------------------------------------------------- profiling
// Eager (non-graph) runs can time every launch with CUDA events on the
// launching stream and charge it the ALGORITHMIC bytes it must move
// (weights + activations + KV it reads/writes once).  bench.py reads this
// to report the dominant kernel's achieved bandwidth.
enum ProfKind { PK_GEMM, PK_ATTN, PK_ROW, PK_MISC, PK_N };
struct ProfRec {
    int kind;
    double wb, tc;  // algorithmic bytes = wb + T * tc (attention: from the KV extents; wb < 0: combine)
    cudaEvent_t a, b;
};
static bool g_prof = false;
static std::vector<ProfRec> g_prof_pending;
static double g_prof_acc[PK_N][3];  // launches, ms, bytes

#define PROF(kind, wb, tc, ...)                            \
    do {                                                   \
        if (g_prof) {                                      \
            ProfRec r__{kind, wb, tc, nullptr, nullptr};   \
            CUDA_OK(cudaEventCreate(&r__.a));              \
            CUDA_OK(cudaEventCreate(&r__.b));              \
            CUDA_OK(cudaEventRecord(r__.a, st));           \
            __VA_ARGS__;                                   \
            CUDA_OK(cudaEventRecord(r__.b, st));           \
            g_prof_pending.push_back(r__);                 \
        } else {                                           \
            __VA_ARGS__;                                   \
        }                                                  \
    } while (0)

void profile_enable(bool on) {
    g_prof = on;
    if (on)
        for (auto& r : g_prof_acc) r[0] = r[1] = r[2] = 0.0;
}
void profile_read(double* out, int kinds) {
    for (int k = 0; k < kinds && k < PK_N; ++k)
        for (int j = 0; j < 3; ++j) out[k * 3 + j] = g_prof_acc[k][j];
}

// One-time kernel attributes (must run before any CUDA-graph capture).
void prepare_fast_kernels() {
    static bool done = false;
    if (done) return;
    attention_prepare();
    gemm_prepare();
    done = true;
}

// Forward over a device-described batch of <= 256 tokens: tokens / plans in
// ws.d_tokens / ws.d_plans (offset t0), ragged descriptors in `db`.  Every
// launch has a fixed grid sized from the host-side upper bounds and reads
// the true token count from device memory, so the sequence is CUDA-graph
// capturable.
void forward_fast_dev(const Model& m, Cache& c, Workspace& ws, const DeviceBatch& db, int t0, bool want_logits,
                      cudaStream_t st) {
    prepare_fast_kernels();
    FastWorkspace* f = ensure_fast(m, c, ws);
    const Config& cfg = m.cfg;
    const int h = cfg.hidden(), mm = cfg.mlp(), heads = cfg.num_heads, hd = cfg.head_dim;
    const int n = db.T_upper;
    SD_CHECK(n <= kChunkTokens, INTERNAL, "device batch larger than one forward chunk");
    const int32_t* tokens = ws.d_tokens + t0;
    const Plan* dplans = ws.d_plans + t0;
    float* resid = ws.d_resid + (size_t)t0 * h;
    int64_t launches = 0;

    GemmArgs base{};
    base.arg_v = f->arg_v;
    base.arg_i = f->arg_i;
    // every GEMM call site owns a counter region, zeroed once per forward
    CUDA_OK(cudaMemsetAsync(f->gemm_cnt, 0, sizeof(int) * ((size_t)f->n_sites * kGemmCntInts + 256), st));
    int* attn_work = f->gemm_cnt + (size_t)f->n_sites * kGemmCntInts;  // one item counter per layer
    auto site = [&](int l, int k) { return f->gemm_cnt + (size_t)(l * 4 + k) * kGemmCntInts; };
    base.h = h;
    base.hd = hd;
    base.heads = heads;
    base.B = c.B;
    base.cap = c.cap;
    base.plans = dplans;
    base.kv = (__nv_bfloat16*)c.kv;

    PROF(PK_ROW, 0.0, 6.0 * h, launch_k(k_embed_ln, dim3(n), dim3(kRowThreads), 0, st, (const __nv_bfloat16*)m.tok16,
                          (const __nv_bfloat16*)m.pos16, tokens, dplans, h, resid, (const float*)m.layers[0].ln1_g,
                          (const float*)m.layers[0].ln1_b, f->xb, (const int*)db.dT));
    launches++;
    AttnArgs at{};
    at.q = f->q;
    at.kv = (const __nv_bfloat16*)c.kv;
    at.plans = dplans;
    at.segs = db.segs;
    at.qidx = db.qidx;
    at.pad = c.layout == PADDED ? c.d_pad : nullptr;
    at.ctx = f->ctx;
    at.part_o = f->part_o;
    at.part_ml = f->part_ml;
    at.cnt = f->attn_cnt;
    at.h = h;
    at.heads = heads;
    at.B = c.B;
    at.cap = c.cap;
    at.max_splits = f->max_splits;
    at.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
    const int splits = std::max(1, (db.max_kv_upper + kAttnSplit - 1) / kAttnSplit);
    const int qtiles = std::max(1, (db.max_q_upper + kAttnQT - 1) / kAttnQT);

    // the four GEMMs of a layer and the LM head, as chain links
    auto qkv = [&](int l, GemmChain& ch, const GemmMaps*& mp) {
        GemmArgs& g = ch.g[ch.n];
        g = base;
        g.epi = EPI_QKV;
        g.M = 3 * h;
        g.K = h;
        g.m_tiles = (3 * h + kGemmTile - 1) / kGemmTile;
        g.cnt = site(l, 0);
        g.bias = m.layers[l].bqkv;
        g.out_bf16 = f->q;
        g.layer = l;
        mp = &f->map_qkv[l];
    };
    auto o_proj = [&](int l, GemmChain& ch, const GemmMaps*& mp) {
        GemmArgs& g = ch.g[ch.n];
        g = base;
        g.epi = EPI_RESID_LN;  // residual, fused with LN2 -> xb
        g.M = h;
        g.K = h;
        g.m_tiles = (h + kGemmTile - 1) / kGemmTile;
        g.cnt = site(l, 1);
        g.bias = m.layers[l].bo;
        g.out_f32 = resid;
        g.ld_out = h;
        g.ln_g = m.layers[l].ln2_g;
        g.ln_b = m.layers[l].ln2_b;
        g.ln_out = f->xb;
        mp = &f->map_o[l];
    };
    auto fc = [&](int l, GemmChain& ch, const GemmMaps*& mp) {
        GemmArgs& g = ch.g[ch.n];
        g = base;
        g.epi = EPI_GELU;
        g.M = mm;
        g.K = h;
        g.m_tiles = (mm + kGemmTile - 1) / kGemmTile;
        g.cnt = site(l, 2);
        g.bias = m.layers[l].bfc;
        g.out_bf16 = f->act;
        g.ld_out = mm;
        mp = &f->map_fc[l];
    };
    auto proj = [&](int l, GemmChain& ch, const GemmMaps*& mp) {
        GemmArgs& g = ch.g[ch.n];
        g = base;
        g.epi = EPI_RESID_LN;  // residual, fused with the next LN1 (or the final LN) -> xb
        g.M = h;
        g.K = mm;
        g.m_tiles = (h + kGemmTile - 1) / kGemmTile;
        g.cnt = site(l, 3);
        g.bias = m.layers[l].bproj;
        g.out_f32 = resid;
        g.ld_out = h;
        g.ln_g = l + 1 < cfg.num_layers ? m.layers[l + 1].ln1_g : m.lnf_g;
        g.ln_b = l + 1 < cfg.num_layers ? m.layers[l + 1].ln1_b : m.lnf_b;
        g.ln_out = f->xb;
        mp = &f->map_proj[l];
    };
    auto lm = [&](GemmChain& ch, const GemmMaps*& mp) {
        GemmArgs& g = ch.g[ch.n];
        g = base;
        g.epi = EPI_ARGMAX;
        g.M = m.vocab_pad;
        g.K = h;
        g.m_tiles = m.vocab_pad / kGemmTile;
        g.cnt = site(cfg.num_layers, 0);
        g.vocab = cfg.vocab_size;
        g.argmax = ws.d_argmax + t0;
        g.logits = want_logits ? ws.d_logits + (size_t)t0 * cfg.vocab_size : nullptr;
        g.flag = ws.d_flag;
        mp = &f->map_lm;
    };
    // algorithmic bytes of a link: weights once + token operand + outputs
    auto link_bytes = [&](const GemmArgs& g, double& wb, double& tc) {
        wb += (double)g.M * g.K * 2;
        double out = g.epi == EPI_QKV ? 3.0 * h * 2 : g.epi == EPI_GELU ? mm * 2.0 : g.epi == EPI_ARGMAX ? 4.0 : h * 10.0;
        tc += g.K * 2.0 + out;
    };
    auto run_chain = [&](GemmChain& ch, const GemmMaps* const* mps) {
        ch.T = n;
        ch.dT = db.dT;
        ch.T_upper = n;
        static const int dbg = getenv("SD_GEMM_DBG") ? atoi(getenv("SD_GEMM_DBG")) : 0;
        ch.dbg = dbg;
        static const int pf = getenv("SD_GEMM_PREFETCH") ? atoi(getenv("SD_GEMM_PREFETCH")) : 0;
        ch.prefetch = pf;
        double wb = 0, tc = 0;
        for (int i = 0; i < ch.n; ++i) {
            ch.g[i].part = f->part[i & 1];
            gemm_plan(ch.g[i], kSms);
            link_bytes(ch.g[i], wb, tc);
        }
        PROF(PK_GEMM, wb, tc, chain_launch(ch, mps, st));
        launches++;
    };

    {  // layer 0's QKV (+ scatter into the arena) on its own
        GemmChain ch{};
        const GemmMaps* mps[kMaxChain];
        qkv(0, ch, mps[0]);
        ch.n = 1;
        run_chain(ch, mps);
    }
    for (int l = 0; l < cfg.num_layers; ++l) {
        // ragged attention of layer l
        at.layer = l;
        at.work = attn_work + l;
        static const int adbg = getenv("SD_ATTN_DBG") ? atoi(getenv("SD_ATTN_DBG")) : 0;
        at.dbg = adbg;
        // split-grid attention with in-kernel split fold (default); SD_ATTN_IMPL=2
        // selects the experimental persistent TMA-ring kernel (attention_sm100.cu)
        static const int aimpl = getenv("SD_ATTN_IMPL") ? atoi(getenv("SD_ATTN_IMPL")) : 1;
        if (aimpl != 2)
            PROF(PK_ATTN, 0.0, 0.0, attention_v1_launch(at, hd, db.max_kv_upper, db.max_q_upper, n, db.dT, st));
        else
            PROF(PK_ATTN, 0.0, 0.0, attention_launch(at, f->kv_map, hd, splits, qtiles, st));
        launches++;
        // one persistent launch: O -> FC -> PROJ -> next layer's QKV (or the LM head)
        GemmChain ch{};
        const GemmMaps* mps[kMaxChain];
        o_proj(l, ch, mps[ch.n]);
        ch.n++;
        fc(l, ch, mps[ch.n]);
        ch.n++;
        proj(l, ch, mps[ch.n]);
        ch.n++;
        if (l + 1 < cfg.num_layers)
            qkv(l + 1, ch, mps[ch.n]);
        else
            lm(ch, mps[ch.n]);
        ch.n++;
        run_chain(ch, mps);
    }
    note_launches(launches);
    CUDA_OK(cudaGetLastError());
    if (g_prof) {  // charge every timed launch its algorithmic bytes
        CUDA_OK(cudaStreamSynchronize(st));
        int T = 0;
        CUDA_OK(cudaMemcpy(&T, db.dT, 4, cudaMemcpyDeviceToHost));
        std::vector<SampleSeg> segs(c.B);
        CUDA_OK(cudaMemcpy(segs.data(), db.segs, sizeof(SampleSeg) * c.B, cudaMemcpyDeviceToHost));
        double kv = 0;
        for (auto& sg : segs) kv += (double)sg.kv_len * (sg.n_q > 0);
        const double attn_bytes = kv * 2 * hd * 2 * heads + (double)T * h * 4;
        for (auto& r : g_prof_pending) {
            float ms = 0.0f;
            CUDA_OK(cudaEventElapsedTime(&ms, r.a, r.b));
            g_prof_acc[r.kind][0] += 1;
            g_prof_acc[r.kind][1] += ms;
            // attention bytes are charged once per layer (the combine adds none)
            g_prof_acc[r.kind][2] += r.kind == PK_ATTN ? (r.wb < 0 ? 0.0 : attn_bytes) : r.wb + (double)T * r.tc;
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        g_prof_pending.clear();
    }
}

// Forward over host-known plans (any T): chunks of <= 256 tokens with ragged
// descriptors built on the host.  Chunking is exact because each sample's
// tokens carry increasing slots and every token only attends to slots <= its
// own, all of which an earlier chunk (or this one) has already written.
void forward_fast(const Model& m, Cache& c, Workspace& ws, int T, bool want_logits, cudaStream_t st) {
    std::vector<Plan> plans(T);
    CUDA_OK(cudaMemcpyAsync(plans.data(), ws.d_plans, sizeof(Plan) * T, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    for (int t0 = 0; t0 < T; t0 += kChunkTokens) {
        int n = std::min(kChunkTokens, T - t0);
        std::vector<SampleSeg> segs(c.B, SampleSeg{0, 0, 0, 0});
        std::vector<std::vector<int>> per(c.B);
        for (int i = 0; i < n; ++i) per[plans[t0 + i].sample].push_back(i);
        std::vector<int32_t> qidx;
        int max_kv = 0, max_q = 0;
        for (int s = 0; s < c.B; ++s) {
            segs[s].q_start = (int)qidx.size();
            segs[s].n_q = (int)per[s].size();
            for (int i : per[s]) {
                qidx.push_back(i);
                segs[s].kv_len = std::max(segs[s].kv_len, plans[t0 + i].write_slot + 1);
            }
            max_kv = std::max(max_kv, segs[s].kv_len);
            max_q = std::max(max_q, segs[s].n_q);
        }
        CUDA_OK(cudaMemcpyAsync(ws.d_segs, segs.data(), sizeof(SampleSeg) * c.B, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemcpyAsync(ws.d_qidx, qidx.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemcpyAsync(ws.d_T, &n, sizeof(int), cudaMemcpyHostToDevice, st));
        DeviceBatch db{ws.d_segs, ws.d_qidx, ws.d_T, n, max_kv, max_q};
        forward_fast_dev(m, c, ws, db, t0, want_logits, st);
        CUDA_OK(cudaStreamSynchronize(st));  // host vectors above are reused per chunk
    }
}

}  // namespace sdb
