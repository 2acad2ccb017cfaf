// Device argument block of one verify step (all pointers are device memory).
#pragma once
#include "common.h"

namespace sdb {

struct StepArgs {
    int B, cap, layout, stop_on_eos, acc_stride;
    // the paper's 2x2 ablation: 0 = as the layout says
    // (unpad: unpadded input + KV; padded: padded input + KV); 1 = unpadded
    // input over the padded KV grid; 2 = padded input (PAD spectators) over
    // the unpadded KV arena
    int ablation;
    // inputs (host-driven step) ----------------------------------------------
    const int32_t* last;     // [B] tokens.back(); null in device mode (read from ctx)
    int32_t* counts;         // [B] draft counts k_s (written by the device predictor)
    int32_t* drafts;         // host mode: concatenated; device mode: [B][kcap]
    int draft_stride;        // 0 = concatenated (host mode), else per-sample stride
    const int32_t* budget;   // [B] max_new_tokens - generated; null in device mode
    int32_t* active;         // [B]
    // device-resident loop state (null in the host-driven step) --------------
    int32_t* ctx;            // [B][ctx_cap] prompt + generated tokens
    int32_t* ctx_len;        // [B]
    int ctx_cap;
    int32_t* gen;            // [B] tokens generated so far
    int max_new;
    int32_t* n_active;       // scalar: samples still active after this step
    int32_t* log_k;          // [max_steps][B] step records (or null)
    int32_t* log_tau;
    int32_t* log_drafts;     // [max_steps][B][log_kcap] the drafts each step verified (or null)
    int log_kcap;
    int32_t* step;           // scalar step counter
    int max_steps;
    // cache descriptors (mutated by k_accept) --------------------------------
    int32_t* committed;      // [B]
    int32_t* logical;        // [B]
    uint8_t* pad;            // [B*cap] or null (unpad)
    // pack outputs / scratch -------------------------------------------------
    int32_t* tokens;         // [T_max]
    Plan* plans;             // [T_max]
    SampleSeg* segs;         // [B]
    int32_t* qidx;           // [T_max]
    int32_t* first_row;      // [B]
    int32_t* draft_off;      // [B]
    int32_t* scalars;        // [0]=T [1]=k_max [2]=grid base [3]=tau_max
    // forward output
    const int32_t* argmax;   // [T_max]
    // accept outputs
    int32_t* tau;            // [B]
    int32_t* accepted;       // [B][acc_stride]
    int32_t* clipped;        // [B]
    // device loop as ONE CUDA-graph WHILE node: k_accept sets the loop
    // condition (samples still active) -- no host round trip, no idle steps
    unsigned long long cond;  // cudaGraphConditionalHandle
    int has_cond;
};

// Device predictors for the resident loop (predictors.cpp:39-72 on device).
struct PredictArgs {
    int kind;                // 1 retrieval (LLMA prompt lookup), 2 synthetic trajectory
    int match_len, copy_len, k, vocab;
    uint64_t seed;
    int id_base;             // global id of local sample 0 (mix_seed uses global ids)
    double accuracy;
    const int32_t* traj;     // [B][traj_stride] greedy continuation (synthetic)
    int traj_stride;
};

// Device draft-model rollout (predictors.cpp:9-37) with a PERSISTENT per-sample
// draft KV cache: the reference re-prefills the whole context on every call;
// here only the 1-2 context tokens the draft cache has not seen are fed, then
// k-1 single-token steps.  Drafts are identical by prefix purity
// (model.hpp:54-57): a token's output depends only on its own prefix.
struct DraftArgs {
    int B, k, kcap, cap;        // draft length, drafts stride, draft-cache capacity
    const int32_t* active;      // [B] target-loop active flags (start of the step)
    const int32_t* ctx;         // [B][ctx_cap] accepted context
    const int32_t* ctx_len;     // [B]
    int ctx_cap;
    int32_t* dcommit;           // [B] draft-cache positions holding context KV
    int32_t* lsnap;             // [B] context length when this step's rollout began
    int32_t* drafts;            // [B][kcap] -> the target verify step
    int32_t* counts;            // [B]
    const int32_t* tau;         // [B] target accept output (commit)
    // the draft forward's ragged batch (the draft cache's workspace)
    int32_t* tokens;
    Plan* plans;
    SampleSeg* segs;
    int32_t* qidx;
    int32_t* dT;
    const int32_t* argmax;      // draft greedy_next per row
};
void launch_draft_pack(const DraftArgs& d, int j, cudaStream_t st);
void launch_draft_take(const DraftArgs& d, int j, cudaStream_t st);
void launch_draft_commit(const DraftArgs& d, cudaStream_t st);

void launch_pack(const StepArgs& a, cudaStream_t st);
void launch_accept(const StepArgs& a, cudaStream_t st);
void launch_pad_fill(const StepArgs& a, const Cache& c, cudaStream_t st);
// PaddedGrid::commit_padded's filler rows from the host API: zero K/V rows
// [r0[i], r1) of sample samples[i] (device arrays, n entries) in every layer
void launch_zero_rows(const Cache& c, const int32_t* samples, const int32_t* r0, int n, int r1, cudaStream_t st);
void launch_predict(const StepArgs& a, const PredictArgs& p, cudaStream_t st);

}  // namespace sdb
