// Host interface of the tcgen05 weight-streaming GEMM (gemm_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.h"

namespace sdb {

enum Epilogue { EPI_STORE = 0, EPI_RESID = 1, EPI_GELU = 2, EPI_QKV = 3, EPI_ARGMAX = 4 };

struct GemmArgs {
    int M, K, m_tiles;        // W is [M_pad][K] bf16, m_tiles = ceil(M / 256)
    int T;                    // token count when dT == nullptr
    const int* dT;            // device token count (graph-capturable), or nullptr
    float* ws;                // split-K partials: [2 * grid][256 cols][256 rows] fp32
    int* counters;            // per-tile arrival counters (zeroed, self-resetting)
    const float* bias;        // [M] or nullptr
    float* out_f32;           // EPI_STORE out / EPI_RESID residual stream
    __nv_bfloat16* out_bf16;  // EPI_GELU activations / EPI_QKV queries
    int ld_out;
    // EPI_QKV scatter into the KV arena [L][2][B][heads][cap][hd]
    __nv_bfloat16* kv;
    const Plan* plans;
    int h, hd, heads, B, cap, layer;
    // EPI_ARGMAX (LM head)
    int vocab, ld_part;
    float* part_val;          // [m_tiles][ld_part]
    int* part_idx;
    float* logits;            // optional [T][vocab]
    int* flag;                // non-finite flag
};

struct GemmMaps {
    CUtensorMap A;     // weights, box {64, 256}
    CUtensorMap B[4];  // tokens, boxes {64, 32/64/128/256}
};

CUtensorMap make_tmap_2d(const void* base, int64_t rows, int64_t cols, int box_rows);
void make_b_maps(GemmMaps& maps, const void* x, int64_t rows, int64_t cols);
int gemm_grid(const GemmArgs& a, int T_upper, int sms);
void gemm_prepare();  // one-time kernel attributes (before any graph capture)
void gemm_launch(int epi, const GemmArgs& a, const GemmMaps& maps, int grid, cudaStream_t st);

}  // namespace sdb
