// Host interface of the ragged verify-step attention (attention_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.h"

namespace sdb {

struct AttnArgs {
    const __nv_bfloat16* q;    // [T][h] queries of the packed stream
    const __nv_bfloat16* kv;   // arena [L][K|V][B][heads][cap][hd]
    const Plan* plans;         // per token: sample, write slot (= causal limit)
    const SampleSeg* segs;     // per sample: query range in qidx, visible KV extent
    const int32_t* qidx;
    const uint8_t* pad;        // padded-grid hole flags [B][cap] or null (unpadded)
    __nv_bfloat16* ctx;        // [T][h] attention output
    float* part_o;             // contributor partials [T][heads][max_splits * 4][hd]
    float* part_ml;            // [T][heads][max_splits * 4][2] (running max, sum)
    int* cnt;                  // [B * heads * kMaxQTiles] split arrival counters (self-resetting)
    int* work;                 // this launch's item counter (zero before the launch)
    int h, heads, B, cap, layer, max_splits;
    int dbg;                   // probe only: bit0 = stream K/V without computing
    float scale_log2;          // log2(e) / sqrt(hd)
};

constexpr int kAttnChunk = 64;     // keys per pipeline stage
constexpr int kAttnSplit = 512;    // keys per work item (split): 8 chunks, two per compute warp
constexpr int kAttnQT = 8;         // queries per work item (the mma N side)
constexpr int kMaxQTiles = 32;     // 256 tokens / 8

// TMA map over the KV arena viewed as [L*2*B*heads*cap rows][hd] bf16, box {64, 64}
CUtensorMap make_kv_map(const void* kv, int64_t rows, int hd);
// one launch: every (sample, head, query tile, split) item of layer a.layer
void attention_launch(const AttnArgs& a, const CUtensorMap& kv_map, int hd, int splits, int qtiles,
                      cudaStream_t st);
void attention_prepare();
// previous generation (attention_v1.cu): grid of split CTAs + combine kernel
void attention_v1_launch(const AttnArgs& a, int hd, int max_kv_upper, int max_q_upper, int T_upper, const int* dT,
                         cudaStream_t st);

}  // namespace sdb
