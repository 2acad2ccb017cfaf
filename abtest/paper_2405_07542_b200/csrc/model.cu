// Weight storage and the counter-mode SplitMix64 initializer.
//
// Model::init (model.cpp:120-139) draws every weight from ONE SplitMix64
// stream (rng.hpp:15-35) in declaration order.  SplitMix64's state after i
// draws is seed + i*gamma, so draw i is a pure function of (seed, i): each
// thread computes its own element independently, bit-identical to the
// sequential CPU loop, and 13B draws take milliseconds instead of minutes
// (SURVEY.md §8a row a18).
#include <cuda_bf16.h>

#include "common.h"

namespace sdb {

void* dmalloc(size_t bytes) {
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    CUDA_OK(cudaMalloc(&p, bytes));
    return p;
}
void dfree(void* p) {
    if (p) cudaFree(p);
}

void WeightLayout::build(const Config& c) {
    int64_t h = c.hidden(), m = c.mlp(), at = 0;
    auto take = [&](int64_t n) {
        int64_t o = at;
        at += n;
        return o;
    };
    tok = take((int64_t)c.vocab_size * h);
    pos = take((int64_t)c.max_positions * h);
    layer.resize(c.num_layers);
    for (auto& o : layer) {
        o.ln1_g = take(h); o.ln1_b = take(h);
        o.wq = take(h * h); o.bq = take(h);
        o.wk = take(h * h); o.bk = take(h);
        o.wv = take(h * h); o.bv = take(h);
        o.wo = take(h * h); o.bo = take(h);
        o.ln2_g = take(h); o.ln2_b = take(h);
        o.w_fc = take(m * h); o.b_fc = take(m);
        o.w_proj = take(h * m); o.b_proj = take(h);
    }
    lnf_g = take(h);
    lnf_b = take(h);
    lm = take((int64_t)c.vocab_size * h);
    total = at;
}

Model::~Model() {
    free_fast_model(fast);
    for (void* p : allocations) dfree(p);
}

Cache::~Cache() {
    dfree(kv);
    dfree(d_committed);
    dfree(d_logical);
    dfree(d_pad);
}

namespace {

__device__ __forceinline__ float draw(uint64_t seed, uint64_t index, float limit) {
    // state after (index+1) next_u64 calls, then the SplitMix64 finalizer
    uint64_t z = seed + (index + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    float u = __fmul_rn((float)(z >> 40), 0x1.0p-24f);   // rng.hpp:23-25
    return __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), limit);  // rng.hpp:33-35
}

// dst[i] = draw(stream_base + i) for i < n
__global__ void k_draw_f32(float* dst, int64_t n, uint64_t seed, uint64_t stream_base, float limit) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = draw(seed, stream_base + (uint64_t)i, limit);
}
__global__ void k_draw_bf16(__nv_bfloat16* dst, int64_t n, uint64_t seed, uint64_t stream_base,
                            float limit) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __float2bfloat16_rn(draw(seed, stream_base + (uint64_t)i, limit));
}
__global__ void k_fill_f32(float* dst, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = v;
}
__global__ void k_f32_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __float2bfloat16_rn(src[i]);
}

int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

float xavier(int fan_in, int fan_out) {  // model.cpp:80-82 (sqrtf is correctly rounded)
    return sqrtf(6.0f / (float)(fan_in + fan_out));
}

// One drawn tensor of Model::init, in stream order.
struct Draw {
    int64_t n;
    float limit;
};

}  // namespace

void init_weights_fp32(Model& m, cudaStream_t st) {
    const Config& c = m.cfg;
    const WeightLayout& L = m.lay;
    int h = c.hidden(), mm = c.mlp();
    float* w = m.w32;
    uint64_t s = c.init_seed, at = 0;
    auto drawn = [&](int64_t off, int64_t n, float limit) {
        k_draw_f32<<<grid_for(n), 256, 0, st>>>(w + off, n, s, at, limit);
        at += (uint64_t)n;
    };
    auto fill = [&](int64_t off, int64_t n, float v) {
        k_fill_f32<<<grid_for(n), 256, 0, st>>>(w + off, n, v);
    };
    drawn(L.tok, (int64_t)c.vocab_size * h, 0.1f);
    drawn(L.pos, (int64_t)c.max_positions * h, 0.1f);
    for (const LayerOff& o : L.layer) {
        fill(o.ln1_g, h, 1.0f); fill(o.ln1_b, h, 0.0f);
        fill(o.ln2_g, h, 1.0f); fill(o.ln2_b, h, 0.0f);
        fill(o.bq, h, 0.0f); fill(o.bk, h, 0.0f); fill(o.bv, h, 0.0f); fill(o.bo, h, 0.0f);
        fill(o.b_fc, mm, 0.0f); fill(o.b_proj, h, 0.0f);
        drawn(o.wq, (int64_t)h * h, xavier(h, h));
        drawn(o.wk, (int64_t)h * h, xavier(h, h));
        drawn(o.wv, (int64_t)h * h, xavier(h, h));
        drawn(o.wo, (int64_t)h * h, xavier(h, h));
        drawn(o.w_fc, (int64_t)mm * h, xavier(h, mm));
        drawn(o.w_proj, (int64_t)h * mm, xavier(mm, h));
    }
    fill(L.lnf_g, h, 1.0f);
    fill(L.lnf_b, h, 0.0f);
    drawn(L.lm, (int64_t)c.vocab_size * h, xavier(h, c.vocab_size));
    CUDA_OK(cudaGetLastError());
}

void init_weights_bf16(Model& m, cudaStream_t st) {
    const Config& c = m.cfg;
    int64_t h = c.hidden(), mm = c.mlp();
    uint64_t s = c.init_seed, at = 0;
    auto drawn = [&](uint16_t* dst, int64_t n, float limit) {
        k_draw_bf16<<<grid_for(n), 256, 0, st>>>((__nv_bfloat16*)dst, n, s, at, limit);
        at += (uint64_t)n;
    };
    auto fill = [&](float* dst, int64_t n, float v) {
        k_fill_f32<<<grid_for(n), 256, 0, st>>>(dst, n, v);
    };
    drawn(m.tok16, (int64_t)c.vocab_size * h, 0.1f);
    drawn(m.pos16, (int64_t)c.max_positions * h, 0.1f);
    for (FastLayer& f : m.layers) {
        fill(f.ln1_g, h, 1.0f); fill(f.ln1_b, h, 0.0f);
        fill(f.ln2_g, h, 1.0f); fill(f.ln2_b, h, 0.0f);
        fill(f.bqkv, 3 * h, 0.0f); fill(f.bo, h, 0.0f); fill(f.bfc, mm, 0.0f); fill(f.bproj, h, 0.0f);
        drawn(f.wqkv, h * h, xavier(h, h));
        drawn(f.wqkv + h * h, h * h, xavier(h, h));
        drawn(f.wqkv + 2 * h * h, h * h, xavier(h, h));
        drawn(f.wo, h * h, xavier(h, h));
        drawn(f.wfc, mm * h, xavier(h, mm));
        drawn(f.wproj, h * mm, xavier(mm, h));
    }
    fill(m.lnf_g, h, 1.0f);
    fill(m.lnf_b, h, 0.0f);
    drawn(m.lm16, (int64_t)c.vocab_size * h, xavier(h, c.vocab_size));
    CUDA_OK(cudaMemsetAsync(m.lm16 + (int64_t)c.vocab_size * h, 0,
                            sizeof(uint16_t) * (size_t)(m.vocab_pad - c.vocab_size) * h, st));
    CUDA_OK(cudaGetLastError());
}

void upload_weights_fp32(Model& m, const float* host, cudaStream_t st) {
    CUDA_OK(cudaMemcpyAsync(m.w32, host, sizeof(float) * (size_t)m.lay.total,
                            cudaMemcpyHostToDevice, st));
}

void upload_weights_bf16(Model& m, const float* host, cudaStream_t st) {
    const Config& c = m.cfg;
    const WeightLayout& L = m.lay;
    int64_t h = c.hidden(), mm = c.mlp();
    // stage each tensor through one fp32 buffer sized for the largest tensor
    int64_t biggest = std::max<int64_t>((int64_t)c.vocab_size * h,
                                        std::max<int64_t>((int64_t)c.max_positions * h, mm * h));
    float* stage = (float*)dmalloc(sizeof(float) * (size_t)biggest);
    auto cvt = [&](uint16_t* dst, int64_t off, int64_t n) {
        CUDA_OK(cudaMemcpyAsync(stage, host + off, sizeof(float) * n, cudaMemcpyHostToDevice, st));
        k_f32_to_bf16<<<grid_for(n), 256, 0, st>>>(stage, (__nv_bfloat16*)dst, n);
        CUDA_OK(cudaStreamSynchronize(st));
    };
    auto f32 = [&](float* dst, int64_t off, int64_t n) {
        CUDA_OK(cudaMemcpyAsync(dst, host + off, sizeof(float) * n, cudaMemcpyHostToDevice, st));
    };
    cvt(m.tok16, L.tok, (int64_t)c.vocab_size * h);
    cvt(m.pos16, L.pos, (int64_t)c.max_positions * h);
    for (int l = 0; l < c.num_layers; ++l) {
        const LayerOff& o = L.layer[l];
        FastLayer& f = m.layers[l];
        f32(f.ln1_g, o.ln1_g, h); f32(f.ln1_b, o.ln1_b, h);
        f32(f.ln2_g, o.ln2_g, h); f32(f.ln2_b, o.ln2_b, h);
        f32(f.bqkv, o.bq, h); f32(f.bqkv + h, o.bk, h); f32(f.bqkv + 2 * h, o.bv, h);
        f32(f.bo, o.bo, h); f32(f.bfc, o.b_fc, mm); f32(f.bproj, o.b_proj, h);
        cvt(f.wqkv, o.wq, h * h);
        cvt(f.wqkv + h * h, o.wk, h * h);
        cvt(f.wqkv + 2 * h * h, o.wv, h * h);
        cvt(f.wo, o.wo, h * h);
        cvt(f.wfc, o.w_fc, mm * h);
        cvt(f.wproj, o.w_proj, h * mm);
    }
    f32(m.lnf_g, L.lnf_g, h);
    f32(m.lnf_b, L.lnf_b, h);
    cvt(m.lm16, L.lm, (int64_t)c.vocab_size * h);
    CUDA_OK(cudaMemsetAsync(m.lm16 + (int64_t)c.vocab_size * h, 0,
                            sizeof(uint16_t) * (size_t)(m.vocab_pad - c.vocab_size) * h, st));
    CUDA_OK(cudaStreamSynchronize(st));
    dfree(stage);
}

}  // namespace sdb
