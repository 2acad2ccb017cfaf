// Opaque handle types behind the C ABI and the host-side operations shared by
// capi.cpp (entry points) and engine.cpp (the decode-loop driver).
#pragma once

#include <memory>

#include "../../include/specdec_b200.h"
#include "../../include/specdec_b200_debug.h"
#include "common.h"
#include "step.h"

struct sd_model {
    sdb::Model m;
    cudaStream_t st = nullptr;
    ~sd_model();
};

// A WriteLedger handle: standalone (sd_ledger_create) or a view of a cache's
// own ledger (sd_cache_ledger_handle; lives and dies with the cache).
struct sd_ledger {
    sdb::Ledger own;
    sdb::Ledger* l = &own;
};

// The host-side half of a verify step enqueued by verify_step_enqueue and
// not yet consumed by verify_step_finish.
struct VerifyInflight {
    bool on = false;
    int kmax = 0, base = 0, K1 = 0;
    size_t o_tau = 0, o_clip = 0, o_acc = 0, o_flag = 0;
    std::vector<int32_t> counts, active;
};

struct sd_cache {
    sdb::Cache c;
    sd_model* model = nullptr;  // null for a dims-only arena until a forward binds a model
    int device = 0;
    int precision = 0;          // element type of the arena (sd_precision)
    sd_ledger lh;               // lh.l -> c.ledger
    bool kv_stored = false;     // a write_kv stored K/V bytes (a dims-only arena can no longer re-lay out)
    cudaStream_t user_stream = nullptr;  // sd_cache_set_stream: all of this cache's work is ordered on it
    cudaEvent_t done_ev = nullptr;       // end of the in-flight verify step
    VerifyInflight inflight;
    sdb::Workspace ws;
    // verify-step device buffers
    int kcap = 0;                 // drafts per sample the buffers hold
    int32_t* d_step = nullptr;    // inputs + scratch + outputs, one allocation
    int32_t* h_step = nullptr;    // pinned host mirror for the H2D / D2H copies
    size_t step_words = 0;
    // sd_verify_step's CUDA graph (pack -> forward -> accept with device-side
    // token counts), rebuilt when any buffer it bakes in changes
    cudaGraphExec_t vgraph = nullptr;
    const void* vg_key[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int vg_flags = -1;
    int vg_calls = 0;
    ~sd_cache();
};

namespace sdb {

void note_launches(int64_t n);
void set_device(int device);

// Host-validated forward over planned tokens (model.cpp:256-373 contract).
// tokens / plans are host arrays of length n.  Mutates the cache exactly like
// the reference (KV writes, ledger, written extent) and optionally returns
// logits [n][V] and argmax [n].
void forward_planned_host(sd_model* m, sd_cache* c, const int32_t* tokens, const Plan* plans, int n,
                          float* logits, int32_t* argmax);

// Ragged forward (model.cpp:235-254): validates slots against the cache.
void forward_ragged_host(sd_model* m, sd_cache* c, const int32_t* tokens, const int32_t* counts,
                         int batch, const int32_t* slot_sample, const int32_t* slot_pos,
                         float* logits, int32_t* argmax);

// One verify step (see sd_verify_step).  accepted has stride kmax+1 where
// kmax = max active draft count; returns that kmax.
int verify_step_host(sd_model* m, sd_cache* c, const int32_t* last, const int32_t* counts,
                     const int32_t* drafts, const int32_t* budget, const int32_t* active,
                     int stop_on_eos, int32_t* tau, int32_t* accepted, int32_t* clipped,
                     float* logits);

void commit_accepted_host(sd_cache* c, int sample, int tau);
void commit_prefill_host(sd_cache* c, const int32_t* samples, const int32_t* lens, int n);
void mark_hole_host(sd_cache* c, int sample, int pos);
int decode_impl(const sd_engine_config& e, sd_model* target, sd_model* draft, const int32_t* prompts,
                const int32_t* prompt_lens, int32_t* gen_tokens, int32_t* gen_counts, int32_t* rec,
                int64_t rec_cap, int64_t* n_rec, int64_t* ledger, double* timing);
void reset_cache(sd_cache* c);  // back to an empty arena (fresh-cache semantics)
std::vector<int32_t> retrieval_predict(const std::vector<int32_t>& ctx, int match_len, int copy_len);
std::vector<int32_t> draft_predict_fresh(sd_model* draft, const std::vector<int32_t>& ctx, int k);
std::vector<int32_t> synthetic_predict_fresh(sd_model* target, const std::vector<int32_t>& ctx, int k, double accuracy,
                                             uint64_t step_seed);

sd_model* create_model(const Config& cfg, int device, int precision, const float* host_weights);
sd_cache* create_cache(sd_model* m, int batch, int capacity, int layout);
// A model-less arena (CacheArena(num_layers, batch, capacity, kv_dim),
// kv_cache.cpp:78-88): one kv_dim-wide head per slot until a forward binds a
// model, which re-lays the (still unwritten) arena out for its heads.
sd_cache* create_cache_dims(int layers, int batch, int capacity, int kv_dim, int layout, int device, int precision);
void bind_cache(sd_cache* c, sd_model* m);
inline cudaStream_t cache_stream(const sd_cache* c) {
    return c->user_stream ? c->user_stream : c->model ? c->model->st : nullptr;
}
// every call that reads or mutates a cache first checks that no asynchronous
// verify step is still in flight on it (sd_verify_step_async / _wait)
inline void check_idle(const sd_cache* c) {
    if (c->inflight.on)
        throw sdb::Error(sdb::CONTRACT, sdb::prefixed(sdb::CONTRACT, "a verify step is in flight on this cache"));
}
void verify_step_enqueue(sd_model* mh, sd_cache* h, const int32_t* last, const int32_t* counts,
                         const int32_t* drafts, const int32_t* budget, const int32_t* active, int stop_on_eos,
                         float* logits, cudaStream_t st);
int verify_step_finish(sd_cache* h, int32_t* tau, int32_t* accepted, int32_t* clipped);

// forward for the bf16 performance mode (fast_kernels.cu)
void forward_fast(const Model& m, Cache& c, Workspace& ws, int T, bool want_logits, cudaStream_t st);
void forward_fast_dev(const Model& m, Cache& c, Workspace& ws, const DeviceBatch& db, int t0, bool want_logits,
                      cudaStream_t st);
void prepare_fast_kernels();
// allocate the bf16 forward's buffers now (not lazily inside a graph capture)
void ensure_fast_workspace(const Model& m, Cache& c, Workspace& ws);
void profile_enable(bool on);
bool profile_on();
void profile_read(double* out, int kinds);

}  // namespace sdb
