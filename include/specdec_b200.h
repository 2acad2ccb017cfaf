/* specdec_b200.h — C ABI of the B200-native EMS-SD verify step.
 *
 * Drop-in boundary for the reference `specdec` library's hot path
 * (/root/reference/proj, C++20).  The reference has no FFI of its own; these
 * are the entry points its callers (engine.cpp decode loop, predictors,
 * tests) bind today, flattened to plain pointers and sizes.  Each function
 * names the reference interface it replaces.
 *
 * Conventions
 *  - Every function returns an sd_status.  On failure sd_last_error() holds a
 *    thread-local message with the reference's prefixes ("config: ",
 *    "capacity: ", "contract: ", "io: ").  Validation happens on the host
 *    BEFORE any state is mutated, as in the reference (kv_cache.cpp:241-294).
 *  - Host buffers unless the name ends in _device; logits are fp32 [T][V].
 *  - A model handle is read-only after creation and may be shared by caches on
 *    its device; a cache handle is single-writer.
 *  - There is no CPU fallback: every compute call runs CUDA kernels built for
 *    sm_100a, and creating a model without a usable B200 fails with
 *    SD_INTERNAL.
 */
#ifndef SPECDEC_B200_H
#define SPECDEC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SD_OK = 0,
    SD_CONFIG = 1,   /* specdec::ConfigError   (common.hpp:18-20) */
    SD_CAPACITY = 2, /* specdec::CapacityError (common.hpp:23-25) */
    SD_CONTRACT = 3, /* specdec::ContractError (common.hpp:28-30) */
    SD_IO = 4,       /* specdec::IoError       (common.hpp:32-34) */
    SD_INTERNAL = 5  /* specdec::Error / CUDA failure / non-finite logit (model.cpp:368-370) */
} sd_status;

typedef enum {
    SD_FP32_CHECK = 0, /* bit-exact with the CPU reference */
    SD_BF16 = 1        /* performance mode: bf16 weights/KV, fp32 accumulation */
} sd_precision;

typedef enum {
    SD_UNPAD = 0,  /* specdec::UnpadArena  (kv_cache.hpp:105-128) — EMS-SD */
    SD_PADDED = 1  /* specdec::PaddedGrid  (kv_cache.hpp:133-168) — vanilla */
} sd_layout;

/* specdec::ModelConfig (model.hpp:14-25) */
typedef struct {
    int32_t num_layers, num_heads, head_dim, vocab_size, max_positions;
    uint64_t init_seed;
} sd_model_config;

/* specdec::EngineConfig (engine.hpp:21-34); mode 0 greedy, 1 vanilla, 2 ems,
 * and for sd_session_* only the paper's ablation: 3 unpadded
 * input over the padded KV grid, 4 padded input over the unpadded KV arena;
 * predictor 0 draft, 1 retrieval, 2 synthetic. */
typedef struct {
    int32_t mode, predictor, k, match_len, copy_len, batch_size, max_new_tokens, stop_on_eos;
    uint64_t seed;
    double synthetic_accuracy;
    /* global id of local sample 0: a rank holding samples [base, base + B) of
     * a sharded batch seeds the synthetic predictor with the GLOBAL sample id,
     * mix_seed(seed, step, base + s) (engine.cpp:182-185), so its drafts and
     * step records equal the single-process run's */
    int32_t sample_id_base;
} sd_engine_config;

typedef struct sd_model sd_model;
typedef struct sd_cache sd_cache;

const char* sd_last_error(void);
/* number of CUDA kernels this thread's library calls have launched so far */
int64_t sd_kernel_launches(void);
/* Per-launch CUDA-event timing of the bf16 forward (eager runs only; graphs
 * are not instrumented).  sd_profile_read fills out[kinds][3] = {launches,
 * total_ms, algorithmic_bytes} for kinds 0 gemm_qkv, 1 gemm_o, 2 gemm_fc,
 * 3 gemm_proj, 4 gemm_lm (each a whole GEMM stage: streaming kernel + split-K
 * reduction + epilogue), 5 attention, 6 layernorm/embed, 7 misc, 8 the
 * streaming GEMM kernel alone (all classes; weights + token operand bytes). */
int sd_profile_enable(int on);
int sd_profile_read(double* out, int kinds);

/* ---- model --------------------------------------------------------------- */
/* ModelConfig::validate (model.cpp:12-18) */
int sd_config_validate(const sd_model_config* cfg);
/* Model::init (model.cpp:120-139): counter-mode SplitMix64 on the GPU,
 * bit-identical draws to the CPU stream (rng.hpp:15-35). */
int sd_model_init(const sd_model_config* cfg, int device, int precision, sd_model** out);
/* Model::load (model.cpp:195-221), SDCK v1 checkpoint */
int sd_model_load(const char* path, int device, int precision, sd_model** out);
/* Model::save (model.cpp:182-193); fp32 check-mode models only */
int sd_model_save(const sd_model* m, const char* path);
/* Model::weight_checksum (model.cpp:223-233); fp32 check-mode models only */
int sd_model_checksum(const sd_model* m, uint64_t* out);
int sd_model_get_config(const sd_model* m, sd_model_config* out);
int64_t sd_model_weight_bytes(const sd_model* m);
/* Weight access for independent reimplementations in tests (model.hpp:81-87:
 * token_embedding, position_embedding, layer(i), final_ln_gain/bias, lm_head).
 * layer -1 selects the model-level tensors: 0 token_embedding [V][h],
 * 1 position_embedding [P][h], 2 final_ln_gain [h], 3 final_ln_bias [h],
 * 4 lm_head [V][h]; layer i >= 0 selects LayerWeights (model.hpp:27-32) in
 * declaration order: 0 ln1_gain, 1 ln1_bias, 2 wq, 3 bq, 4 wk, 5 bk, 6 wv,
 * 7 bv, 8 wo, 9 bo, 10 ln2_gain, 11 ln2_bias, 12 w_fc, 13 b_fc, 14 w_proj,
 * 15 b_proj (matrices row-major [out][in]).  out receives `count` fp32 values
 * (count must equal the tensor size); a bf16 model returns its stored bf16
 * values widened to fp32. */
int sd_model_get_tensor(const sd_model* m, int layer, int tensor, float* out, int64_t count);
void sd_model_destroy(sd_model* m);

/* ---- KV cache (CacheArena, kv_cache.hpp:65-168) -------------------------- */
int sd_cache_create(const sd_model* m, int batch, int capacity, int layout, sd_cache** out);
/* CacheArena::committed_len / logical_len, UnpadArena::start_offset */
int sd_cache_committed_len(const sd_cache* c, int sample, int32_t* out);
int sd_cache_logical_len(const sd_cache* c, int sample, int32_t* out);
int sd_cache_start_offset(const sd_cache* c, int sample, int32_t* out);
/* UnpadArena::commit_accepted (kv_cache.cpp:152-161): metadata only */
int sd_cache_commit_accepted(sd_cache* c, int sample, int tau);
/* committed_len (and, for the unpad arena, start_offset) of all B samples at
 * once (kv_cache.hpp:109-110); start_offset may be NULL. */
int sd_cache_get_lengths(const sd_cache* c, int32_t* committed, int32_t* start_offset);
/* UnpadArena::commit_accepted for every sample (taus[B]; 0 = not committed),
 * all validated before any state changes. */
int sd_commit_accepted(sd_cache* c, const int32_t* taus);
/* PaddedGrid::commit_padded (kv_cache.cpp:269-314): zero-filler rows on device */
int sd_cache_commit_padded(sd_cache* c, const int32_t* samples, const int32_t* taus, int n);
/* PaddedGrid::commit_prefill (kv_cache.cpp:237-267) */
int sd_cache_commit_prefill(sd_cache* c, const int32_t* samples, const int32_t* lens, int n);
/* CacheArena::mark_hole (kv_cache.cpp:90-92, 215-219) */
int sd_cache_mark_hole(sd_cache* c, int sample, int position);
/* PaddedGrid::is_pad */
int sd_cache_is_pad(const sd_cache* c, int sample, int row, int32_t* out);
/* WriteLedger totals (kv_cache.cpp:44-52) */
int sd_cache_ledger(const sd_cache* c, int64_t* useful, int64_t* padding);
/* Copy visible K/V rows [0, upto] of one (sample, layer) to the host, skipping
 * pad rows — CacheArena::gather_visible (kv_cache.cpp:140-150, 221-235);
 * k_out / v_out are [upto+1][hidden] fp32. */
int sd_cache_gather_visible(const sd_cache* c, int sample, int upto, int layer, float* k_out,
                            float* v_out, int32_t* count);
/* A model-less arena, CacheArena(num_layers, batch, capacity, kv_dim)
 * (kv_cache.hpp:68-73, kv_cache.cpp:78-88): K/V rows can be stored with
 * sd_cache_write_kv and read back with sd_cache_gather_visible; the first
 * forward binds a model of the same depth and width (the arena then takes
 * the model's head split, precision and device, which requires that no row
 * was stored yet if they differ).  precision: SD_FP32_CHECK or SD_BF16. */
int sd_cache_create_dims(int num_layers, int batch, int capacity, int kv_dim, int layout, int device,
                         int precision, sd_cache** out);
/* CacheArena::write_kv (kv_cache.hpp:82-83; kv_cache.cpp:128-138, 203-213):
 * store one token's key and value ([kv_dim] fp32 each; rounded to bf16 in a
 * bf16 arena) for one layer.  The ledger counts the slot once, on layer 0. */
int sd_cache_write_kv(sd_cache* c, int sample, int position, int layer, const float* k_vec,
                      const float* v_vec);
void sd_cache_destroy(sd_cache* c);

/* ---- write ledger (WriteLedger, kv_cache.hpp:13-57) ----------------------- */
/* Useful / padding KV slot writes per sample and the per-step grouping of one
 * decode iteration (begin_step, note_tau per committed sample, end_step).
 * Every cache owns one (sd_cache_ledger_handle, valid while the cache lives):
 * forwards count useful slots, commit_padded counts its filler rows and notes
 * each tau -- it therefore needs an open step, as in the reference -- and
 * sd_verify_step records one whole step (it opens and closes the step itself
 * unless the caller holds one open).  sd_ledger_create makes a standalone
 * WriteLedger(batch). */
typedef struct sd_ledger sd_ledger;
int sd_ledger_create(int batch, sd_ledger** out);
void sd_ledger_destroy(sd_ledger* l); /* no-op for a cache's own ledger */
int sd_cache_ledger_handle(sd_cache* c, sd_ledger** out);
int sd_ledger_note_useful(sd_ledger* l, int sample);
int sd_ledger_note_padding(sd_ledger* l, int sample);
int sd_ledger_begin_step(sd_ledger* l);
int sd_ledger_note_tau(sd_ledger* l, int tau);
int sd_ledger_end_step(sd_ledger* l);
int sd_ledger_batch(const sd_ledger* l, int32_t* batch);
/* useful_total / padding_total (either pointer may be NULL) */
int sd_ledger_totals(const sd_ledger* l, int64_t* useful, int64_t* padding);
/* useful_by_sample / padding_by_sample: [batch] each, either may be NULL */
int sd_ledger_by_sample(const sd_ledger* l, int64_t* useful, int64_t* padding);
int sd_ledger_num_steps(const sd_ledger* l, int64_t* n);
/* LedgerStep i: tau_list (up to cap entries; n_tau = its full length), tau_max,
 * pad_writes, useful_writes */
int sd_ledger_step(const sd_ledger* l, int64_t i, int32_t* tau_list, int32_t cap, int32_t* n_tau,
                   int32_t* tau_max, int64_t* pad_writes, int64_t* useful_writes);
/* WriteLedger::dump_json (kv_cache.cpp:53-62), byte-identical to nlohmann's
 * compact dump; *len = full length, buf gets at most cap-1 bytes + NUL */
int sd_ledger_dump_json(const sd_ledger* l, char* buf, int64_t cap, int64_t* len);
/* padding_ratio (kv_cache.cpp:64-76); SD_CONTRACT when no step was recorded */
int sd_ledger_padding_ratio(const sd_ledger* l, double* out);

/* ---- ragged batching (ragged.cpp:6-36) ----------------------------------- */
int sd_restore_indices(const int32_t* counts, int batch, int flat_index, int32_t* sample,
                       int32_t* position);

/* ---- forward ------------------------------------------------------------- */
/* Model::forward(RaggedBatch, CacheArena&, slots) (model.hpp:71-72,
 * model.cpp:235-254).  tokens are the concatenated inputs, counts the per-sample
 * counts (zero allowed), slot_* the absolute (sample, position) of each token.
 * logits: [T][V] fp32 or NULL; argmax: [T] (greedy_next of each row) or NULL. */
int sd_forward(const sd_model* m, sd_cache* c, const int32_t* tokens, const int32_t* counts,
               int batch, const int32_t* slot_sample, const int32_t* slot_pos, float* logits,
               int32_t* argmax);
/* Model::forward_planned (model.hpp:76-78, model.cpp:256-373) */
int sd_forward_planned(const sd_model* m, sd_cache* c, const int32_t* tokens, int n,
                       const int32_t* sample, const int32_t* logical_pos, const int32_t* write_slot,
                       const int32_t* store, float* logits, int32_t* argmax);

/* ---- fused verify step (engine.cpp:391-489 one iteration) ----------------- */
/* One EMS (or vanilla, by the cache layout) verify step for all B samples:
 * pack [last] + drafts (Algorithm 1) -> forward -> greedy verify (Eq. 5,
 * engine.cpp:60-76) -> budget/EOS clip (engine.cpp:454-463) -> per-sample
 * commit (kv_cache.cpp:152-161 / 269-314).
 *   last_tokens[B]          tokens.back() of each sample
 *   draft_counts[B]         k_s; a sample with active[s]==0 gets no input
 *   drafts                  concatenated drafts, sum(k_s) tokens
 *   budget_left[B]          max_new_tokens - generated
 *   active[B]               0 for finished samples
 * Outputs: tau[B] (0 for inactive), accepted[B][k_max+1], clipped[B],
 * logits (optional, [T][V] in flat token order). */
int sd_verify_step(sd_model* m, sd_cache* c, const int32_t* last_tokens,
                   const int32_t* draft_counts, const int32_t* drafts,
                   const int32_t* budget_left, const int32_t* active, int stop_on_eos,
                   int32_t* tau, int32_t* accepted, int32_t* clipped, float* logits);

/* The same step, asynchronous (calls are stream-ordered and
 * async until outputs are read).  sd_verify_step_async validates on the host
 * (errors are returned before anything is enqueued, nothing mutated), copies
 * the inputs to pinned staging and enqueues H2D -> pack -> forward -> accept
 * [-> pad_fill] -> D2H on `stream` (a cudaStream_t; NULL = the cache's stream,
 * see sd_cache_set_stream), then returns.  sd_verify_step_wait blocks until
 * that work is done, raises device-side errors (non-finite logit) and applies
 * the commit to the cache's host mirrors and ledger; accepted is
 * [B][k_max + 1] with k_max the largest active draft count of that step.
 * Between the two calls every other call on the cache returns SD_CONTRACT.
 * Logits are not available on this path. */
int sd_verify_step_async(sd_model* m, sd_cache* c, const int32_t* last_tokens,
                         const int32_t* draft_counts, const int32_t* drafts,
                         const int32_t* budget_left, const int32_t* active, int stop_on_eos, void* stream);
int sd_verify_step_wait(sd_cache* c, int32_t* tau, int32_t* accepted, int32_t* clipped);
/* Order all of this cache's device work on `stream` (a cudaStream_t; NULL
 * restores the model's internal stream). */
int sd_cache_set_stream(sd_cache* c, void* stream);

/* ---- predictors (predictors.hpp:13-20, predictors.cpp) ------------------- */
/* draft_predict: greedy k-token rollout of `draft` after `context` (a fresh
 * one-sample arena per call); out[k].  ContractError for k < 1 or an empty
 * context, CapacityError when context + k exceeds max_positions. */
int sd_draft_predict(sd_model* draft, const int32_t* context, int n, int k, int32_t* out);
/* retrieval_predict (LLMA prompt lookup): copy <= copy_len tokens that followed
 * the rightmost earlier occurrence of the last match_len tokens; out[copy_len],
 * *n_out tokens written (0 when nothing matches). */
int sd_retrieval_predict(const int32_t* context, int n, int match_len, int copy_len, int32_t* out, int32_t* n_out);
/* synthetic_predict: the target's greedy rollout with each position replaced by
 * (id + 1) % vocab unless a SplitMix64(step_seed) coin lands below accuracy;
 * ConfigError unless 0 <= accuracy < 1; out[k]. */
int sd_synthetic_predict(sd_model* target, const int32_t* context, int n, int k, double accuracy, uint64_t step_seed,
                         int32_t* out);

/* ---- engine (decode_speculative / decode_greedy, engine.cpp:206-489) ------ */
/* prompts: concatenated token ids (BOS included), prompt_lens[B].
 * gen_tokens[B][max_new_tokens], gen_counts[B]; step records as rows of
 * {step, sample, k, tau, clipped, 0} (rec_cap rows max); ledger[2] =
 * {useful_kv_writes, padding_kv_writes}; timing[2] = {prefill_s, decode_s}. */
int sd_decode(const sd_engine_config* cfg, sd_model* target, sd_model* draft,
              const int32_t* prompts, const int32_t* prompt_lens, int32_t* gen_tokens,
              int32_t* gen_counts, int32_t* rec, int64_t rec_cap, int64_t* n_rec,
              int64_t* ledger, double* timing);

/* ---- decode sessions (device-resident decode_speculative loop) ----------- */
/* A session owns one cache and a prefilled batch, and runs the loop of
 * engine.cpp:391-489 entirely on the GPU: the predictor (LLMA retrieval,
 * predictors.cpp:39-59, or the synthetic corrupted greedy rollout,
 * predictors.cpp:61-72, fed from a precomputed trajectory), pack, forward,
 * verify, clip and commit, replayed from a captured CUDA graph.  bf16 models
 * only; cfg->mode 1 (vanilla, padded grid) or 2 (EMS, unpadded arena). */
typedef struct sd_session sd_session;
const char* sd_session_last_error(void);
int sd_session_create(sd_model* m, const sd_engine_config* cfg, int capacity, sd_session** out);
/* draft-model speculative decoding (cfg->predictor 0, predictors.cpp:9-37) on
 * the device: the draft model keeps a persistent per-sample KV cache (the
 * reference re-prefills the whole context per call), feeds only the 1-2
 * context tokens it has not seen, then rolls out cfg->k greedy drafts; rollback
 * after verification is metadata.  Drafts are identical by prefix purity. */
int sd_session_create_draft(sd_model* target, sd_model* draft, const sd_engine_config* cfg, int capacity,
                            sd_session** out);
/* prefill (engine.cpp:330-385) and snapshot the post-prefill state */
int sd_session_prefill(sd_session* s, const int32_t* prompts, const int32_t* prompt_lens);
/* traj[B][stride]: each sample's greedy continuation (synthetic predictor) */
int sd_session_set_trajectory(sd_session* s, const int32_t* traj, int stride);
/* roll back to the post-prefill state (metadata only, no KV moves) */
int sd_session_reset(sd_session* s);
/* run until every sample finished; steps = verify steps, gpu_ms = CUDA-event
 * time on the session stream from the first step to the last */
int sd_session_run(sd_session* s, int use_graph, int graph_steps, int32_t* steps, float* gpu_ms);
/* the same loop driven from the host through sd_verify_step (predictor on the
 * host, H2D drafts / D2H tau + accepted per step); reports the bytes moved */
int sd_session_run_host(sd_session* s, int32_t* steps, float* gpu_ms, int64_t* h2d_bytes, int64_t* d2h_bytes);
/* gen_tokens[B][max_new_tokens], gen_counts[B]; per-step logs [max_steps][B]
 * of draft counts k (-1 inactive) and tau (| 0x10000 when clipped) */
int sd_session_outputs(sd_session* s, int32_t* gen_tokens, int32_t* gen_counts, int32_t* log_k,
                       int32_t* log_tau, int max_steps);
/* the drafts each verify step checked: [max_steps][B][kcap] (kcap = k, or
 * copy_len for the retrieval predictor); entry j < log_k[step][s] is valid */
int sd_session_draft_log(sd_session* s, int32_t* drafts, int max_steps);
int sd_session_cache(sd_session* s, sd_cache** out);
/* run n device steps eagerly (no graph, no completion loop) -- profiling */
int sd_session_step(sd_session* s, int n);
void sd_session_destroy(sd_session* s);

/* ---- multi-GPU: samples sharded over the GPUs of one box */
/* Weights are replicated and every rank runs its own verify loop (global
 * sample ids: sd_engine_config.sample_id_base); the step has no collective.
 * The per-sample outputs are all-gathered once at the end over NCCL
 * (libnccl.so.2, opened at first use).  Bootstrap for C++ hosts: rank 0 calls
 * sd_nccl_unique_id and ships the 128 bytes to every rank out of band; each
 * rank then calls sd_comm_init on its own GPU. */
typedef struct sd_comm sd_comm;
const char* sd_comm_last_error(void);
int sd_nccl_unique_id(uint8_t* id /* [128] */);
int sd_comm_init(const uint8_t* id, int world, int rank, int device, sd_comm** out);
int sd_comm_size(const sd_comm* c, int* world, int* rank);
void sd_comm_destroy(sd_comm* c);
/* every rank sends `count` int32 (same count on all ranks), every rank
 * receives world * count of them in rank order; host buffers */
int sd_comm_allgather_i32(sd_comm* c, const int32_t* local, int64_t count, int32_t* all);
/* A finished session's outputs gathered over all ranks in global sample
 * order (rank r holds samples [r B, (r+1) B)): gen_tokens [world B][max_new],
 * gen_counts [world B]; every rank's session must have the same B and
 * max_new_tokens. */
int sd_session_gather_outputs(sd_session* s, sd_comm* c, int32_t* gen_tokens, int32_t* gen_counts);

#ifdef __cplusplus
}
#endif
#endif /* SPECDEC_B200_H */
