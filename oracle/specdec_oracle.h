/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference `specdec`
 * hot path (EMS unpadded verify step and its padded comparator), used by
 * tests/ as the parity checker and by bench.py's cpu_baseline leg.  It is
 * never linked into or called by the product library.
 *
 * Every function cites the reference file:line (relative to
 * /root/reference/proj) whose algorithm it restates.  Arithmetic order is
 * the reference's and it calls the host libm
 * expf/tanhf/sqrtf exactly as model.cpp does, so on the same host it is
 * bit-identical to the reference; tests/test_oracle.py pins that against the
 * reference itself (oracle/_ref) and the committed golden fixtures.
 *
 * Status codes mirror common.hpp:13-34: 0 ok, 1 Config, 2 Capacity,
 * 3 Contract, 4 Io, 5 other Error. */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t num_layers, num_heads, head_dim, vocab_size, max_positions;
    uint64_t init_seed;
} so_config;

typedef struct so_model so_model;
typedef struct so_cache so_cache;

const char* so_last_error(void);

/* FNV-1a 64 over raw bytes (model.cpp:223-233 hash, reused to fingerprint logits rows) */
uint64_t so_fnv1a(const void* data, int64_t nbytes);

/* rng.hpp:11-46 */
uint64_t so_splitmix_next(uint64_t* state);
uint64_t so_mix_seed(uint64_t a, uint64_t b, uint64_t c);

/* model.cpp:12-18, 91-139, 182-233 */
int so_config_validate(const so_config* c);
int so_model_init(const so_config* c, so_model** out);
int so_model_load(const char* path, so_model** out);
int so_model_save(const so_model* m, const char* path);
void so_model_free(so_model* m);
uint64_t so_model_checksum(const so_model* m);
const float* so_model_weights(const so_model* m, int64_t* count); /* declaration order */
void so_model_get_config(const so_model* m, so_config* out);

/* ragged.cpp:6-36 */
int so_restore_indices(const int32_t* counts, int batch, int flat, int32_t* sample, int32_t* pos);

/* kv_cache.cpp:96-314; layout 0 = UnpadArena, 1 = PaddedGrid */
int so_cache_new(int layout, int layers, int batch, int capacity, int kv_dim, so_cache** out);
void so_cache_free(so_cache* c);
int so_cache_committed(const so_cache* c, int s, int32_t* out);
int so_cache_logical(const so_cache* c, int s, int32_t* out);
int so_cache_start_offset(const so_cache* c, int s, int32_t* out);
int so_cache_commit(so_cache* c, int s, int tau);
int so_cache_commit_padded(so_cache* c, const int32_t* samples, const int32_t* taus, int n);
int so_cache_commit_prefill(so_cache* c, const int32_t* samples, const int32_t* lens, int n);
int so_cache_mark_hole(so_cache* c, int s, int pos);
int so_cache_write_kv(so_cache* c, int s, int pos, int layer, const float* k, const float* v);
int so_cache_gather(const so_cache* c, int s, int upto, int layer, float* k, float* v, int32_t* count);
int64_t so_ledger_useful(const so_cache* c);
int64_t so_ledger_padding(const so_cache* c);

/* model.cpp:235-373.  logits: n x vocab fp32 (nullable), argmax: n (nullable) */
int so_forward(const so_model* m, so_cache* c, const int32_t* tokens, const int32_t* counts,
               int batch, const int32_t* slot_sample, const int32_t* slot_pos, float* logits,
               int32_t* argmax);
int so_forward_planned(const so_model* m, so_cache* c, const int32_t* tokens, int n,
                       const int32_t* sample, const int32_t* logical, const int32_t* slot,
                       const int32_t* store, float* logits, int32_t* argmax);

/* model.cpp:34-41; engine.cpp:60-76 */
int32_t so_greedy_next(const float* row, int vocab);
int so_verify(const float* rows, int nrows, int vocab, const int32_t* drafts, int k,
              int32_t* accepted, int32_t* tau);

/* predictors.cpp:9-72 */
int so_retrieval_predict(const int32_t* ctx, int n, int match_len, int copy_len, int32_t* out,
                         int32_t* nout);
int so_draft_predict(const so_model* draft, const int32_t* ctx, int n, int k, int32_t* out);

/* engine.cpp:291-489: speculative decode (mode 1 vanilla, 2 ems) or greedy (0).
 * prompts: already tokenized incl. BOS, packed with prompt_lens[b].
 * Outputs: gen_tokens [b * max_new], gen_counts [b];
 * step records flattened: per (step, active sample) one row of
 * rec[6] = {step, sample, k, tau, clipped, 0}; n_rec returned;
 * ledger[2] = {useful_writes, padding_writes}.  rec_cap bounds rec rows.
 * predictor: 0 draft, 1 retrieval, 2 synthetic. */
typedef struct {
    int32_t mode, predictor, k, match_len, copy_len, batch_size, max_new_tokens, stop_on_eos;
    uint64_t seed;
    double synthetic_accuracy;
} so_engine_config;

int so_decode(const so_engine_config* cfg, const so_model* target, const so_model* draft,
              const int32_t* prompts, const int32_t* prompt_lens, int32_t* gen_tokens,
              int32_t* gen_counts, int32_t* rec, int64_t rec_cap, int64_t* n_rec,
              int64_t* ledger);

#ifdef __cplusplus
}
#endif
