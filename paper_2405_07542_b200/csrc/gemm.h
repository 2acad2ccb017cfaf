// Host interface of the tcgen05 weight-streaming GEMM chain (gemm_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.h"

namespace sdb {

// What the in-kernel split-K reduction does with the finished sums.
enum Epilogue {
    EPI_STORE = 0,    // out_f32[t][m] = y (+ bias)
    EPI_RESID_LN = 1, // resid[t][m] += y + b; then LayerNorm(resid[t]) -> ln_out (bf16)
    EPI_GELU = 2,     // out_bf16[t][m] = gelu(y + b)
    EPI_QKV = 3,      // Q -> out_bf16, K/V -> KV arena at each token's write slot
    EPI_ARGMAX = 4,   // argmax over the vocab (lowest id on ties) -> argmax[t]
};

constexpr int kGemmTile = 128;        // output features per stream-K tile (one UMMA M=128 accumulator)
constexpr int kGemmCntInts = 1024;    // counter ints per GEMM call site
constexpr int kGemmMaxTiles = 512;    // tiles a call site may have (counter region [0, 512))
constexpr int kMaxChain = 4;          // GEMMs per persistent launch

struct GemmArgs {
    int epi;                  // Epilogue
    int M, K, m_tiles;        // W is [m_tiles * 128][K] bf16 (rows >= M are zero or ignored)
    int max_contrib;          // stream-K schedule (set by gemm_plan)
    int n_slices;             // sum over tiles of their contributor counts (set by gemm_plan)
    int owner_mode;           // 1: each tile's k-block-0 CTA reduces it (few contributors per tile);
                              // 0: every CTA reduces an equal share of all tiles (set by gemm_plan)
    float* part;              // fp32 partial sums [m_tiles * max_contrib][256 tok][128 rows]
    int* cnt;                 // this call site's kGemmCntInts counters, zero before the launch
    const float* bias;        // [M] or nullptr
    float* out_f32;           // EPI_STORE output / EPI_RESID_LN residual stream
    __nv_bfloat16* out_bf16;  // EPI_GELU activations / EPI_QKV queries
    int ld_out;
    const float *ln_g, *ln_b; // EPI_RESID_LN
    __nv_bfloat16* ln_out;
    // EPI_QKV scatter into the KV arena [L][2][B][heads][cap][hd]
    __nv_bfloat16* kv;
    const Plan* plans;
    int h, hd, heads, B, cap, layer;
    // EPI_ARGMAX (LM head)
    int vocab;
    int32_t* argmax;
    float* logits;            // optional [T][vocab]
    int* flag;                // non-finite flag
    float* arg_v;             // [256 tokens][kGemmMaxTiles] per-tile maxima
    int* arg_i;               // [256 tokens][kGemmMaxTiles] their (lowest) ids
};

// Up to kMaxChain dependent GEMMs streamed by ONE persistent launch: GEMM
// i+1's weights stream into the ring while GEMM i is reduced; its token
// operand is loaded once every CTA has finished GEMM i.
struct GemmChain {
    int n;
    int T;                    // token count when dT == nullptr (<= 256)
    const int* dT;            // device token count (graph-capturable), or nullptr
    int T_upper;              // host-side bound (sizes the token tile)
    int sb;                   // token (B) ring depth, 0 = default
    int dbg;                  // probe only: bit0 skip MMAs, bit1 skip partial stores
    int prefetch;             // weight units an idle warp pulls into L2 ahead of the ring (0 = off)
    GemmArgs g[kMaxChain];    // consecutive GEMMs must use different partial buffers
};

struct GemmMaps {
    CUtensorMap A;     // weights, box {64, 128}
    CUtensorMap B[4];  // tokens, boxes {64, 32/64/128/256}
};

CUtensorMap make_tmap_2d(const void* base, int64_t rows, int64_t cols, int box_rows);
void make_b_maps(GemmMaps& maps, const void* x, int64_t rows, int64_t cols);
// fill a.max_contrib / a.n_slices for this shape on `sms` SMs
void gemm_plan(GemmArgs& a, int sms);
// floats the partial buffer needs for a shape (max over the model's GEMMs)
size_t gemm_part_floats(int M, int K, int sms);
// one persistent launch of the chain (B maps chosen from `maps[i].B` by T_upper)
void chain_launch(const GemmChain& c, const GemmMaps* const* maps, cudaStream_t st);
void gemm_prepare();  // one-time kernel attributes (before any graph capture)

}  // namespace sdb
