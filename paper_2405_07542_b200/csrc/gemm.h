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
// LayerNorm rows of the residual stream (a.out_f32, width a.M) -> a.ln_out
void ln_rows_launch(const GemmArgs& a, int T_upper, cudaStream_t st);

// ---- cluster split-K GEMM for small models (gemm_cluster.cu)
struct ClArgs {
    int M, K;                  // W is [M][K] bf16, M % 128 == 0, K % 64 == 0
    int T;                     // token count when dT == nullptr
    const int* dT;             // device token count
    int t_base;                // this launch covers tokens [t_base, t_base + 128)
    int CS, nkb_max, box;      // set by gemm_cl_launch
    int recv_off, per_owner;   // reduction receive buffer offset, tokens each CTA reduces
    const float* bias;         // [M]
    // LN_IN (QKV / FC): the token operand is LayerNorm(x_resid) built in shared memory
    const float* x_resid;      // [T][hidden] fp32 residual stream
    const float2* stats_in;    // [T][n_stat] per-(token, 128-row tile) (sum, M2) of x_resid
    const float *ln_g, *ln_b;
    int hidden, n_stat;        // n_stat = hidden / 128
    // EPI_RESID_LN: resid[t][m] += y + b, then stats_out[t][tile] = (sum, M2) of the new rows
    float* resid;
    float2* stats_out;
    // EPI_GELU activations / EPI_QKV queries
    __nv_bfloat16* out_bf16;
    int ld_out;
    // EPI_QKV scatter into the KV arena [L][2][B][heads][cap][hd]
    __nv_bfloat16* kv;
    const Plan* plans;
    int h, hd, heads, B, cap, layer;
};
struct ClPlan {
    bool ok;
    int CS, nkb_max, tiles, per_owner;
    size_t smem, recv_off;
};
// cluster size / k-blocks per CTA for a shape: a function of (M, K, SMs) only
ClPlan gemm_cl_plan(int M, int K, int box, int sms);
bool gemm_cl_schedulable(const ClPlan& p);
void gemm_cl_prepare();
// epi: EPI_QKV (LN_IN), EPI_GELU (LN_IN) or EPI_RESID_LN (TMA token operand, stats out);
// T_upper <= 128 tokens from a.t_base
void gemm_cl_launch(int epi, const ClArgs& a, const GemmMaps& maps, int T_upper, cudaStream_t st);

}  // namespace sdb
