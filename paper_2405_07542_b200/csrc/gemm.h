// Host interface of the tcgen05 weight-streaming GEMM (gemm_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.h"

namespace sdb {

// What the split-K reduction kernel does with the finished sums.
enum Epilogue {
    EPI_STORE = 0,    // out_f32[t][m] = y
    EPI_RESID_LN = 1, // resid[t][m] += y + b; then LayerNorm(resid[t]) -> ln_out (bf16)
    EPI_GELU = 2,     // out_bf16[t][m] = gelu(y + b)
    EPI_QKV = 3,      // Q -> out_bf16, K/V -> KV arena at each token's write slot
    EPI_ARGMAX = 4,   // argmax over the vocab (lowest id on ties) -> argmax[t]
};

// LM-head argmax scratch: per (token, vocab group) (max, lowest id) partials
// and a self-resetting arrival counter per token.  Owned by the forward's
// workspace (one per cache), never shared between streams or devices.
constexpr int kArgmaxGroups = 64;
struct ArgmaxScratch {
    float* val = nullptr;  // [256][kArgmaxGroups]
    int* idx = nullptr;    // [256][kArgmaxGroups]
    int* cnt = nullptr;    // [256]
};

struct GemmArgs {
    int M, K, m_tiles;        // W is [m_tiles * 256][K] bf16 (zero-padded rows)
    int T;                    // token count when dT == nullptr (must be <= 256)
    const int* dT;            // device token count (graph-capturable), or nullptr
    int grid, max_contrib;    // stream-K schedule (set by gemm_plan)
    int box;                  // token-tile rows staged per k-block (set by gemm_launch)
    float* part;              // fp32 partial sums [m_tiles * max_contrib][256 tok][256 rows]
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
    ArgmaxScratch am;
    int probe;                // 0 in the library; tools/micro probe builds (-DSD_GEMM_PROBE) only
};

struct GemmMaps {
    CUtensorMap A;     // weights, box {64, 256}
    CUtensorMap B[4];  // tokens, boxes {64, 32/64/128/256}
};

CUtensorMap make_tmap_2d(const void* base, int64_t rows, int64_t cols, int box_rows);
void make_b_maps(GemmMaps& maps, const void* x, int64_t rows, int64_t cols);
// fill a.grid / a.max_contrib for this shape on `sms` SMs
void gemm_plan(GemmArgs& a, int sms);
// floats the partial buffer needs for a shape (max over the model's GEMMs)
size_t gemm_part_floats(int M, int K, int sms);
// stream the weights (tcgen05 mainloop -> fp32 partials), then reduce + epilogue
// (`after_stream`, if given, is recorded between the two: profiling)
void gemm_launch(int epi, const GemmArgs& a, const GemmMaps& maps, int T_upper, cudaStream_t st,
                 cudaEvent_t after_stream = nullptr);
void gemm_prepare();  // one-time kernel attributes (before any graph capture)

}  // namespace sdb
