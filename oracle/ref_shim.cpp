// TEST INFRASTRUCTURE ONLY. extern "C" shim over the UNMODIFIED reference
// `specdec` library (compiled in place from /root/reference/proj/src by
// oracle/Makefile). It lets tests/, tests/golden/make_golden.py and the
// `bench.py --impl reference` arm drive the reference through its own public
// API (include/specdec/*.hpp) from Python via ctypes. Nothing here is shipped
// or linked into the product library.
//
// Every entry point returns 0 on success or a nonzero code mirroring the
// reference error taxonomy (common.hpp:13-34): 1 Config, 2 Capacity,
// 3 Contract, 4 Io, 5 other Error / std::exception. The message is kept in a
// thread-local buffer readable with ref_last_error().

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "naive_model.hpp"
#include "specdec/engine.hpp"
#include "specdec/kv_cache.hpp"
#include "specdec/model.hpp"
#include "specdec/predictors.hpp"
#include "specdec/ragged.hpp"
#include "specdec/rng.hpp"

using namespace specdec;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const CapacityError& e) {
        g_err = e.what();
        return 2;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

ModelConfig make_cfg(const int32_t* dims, uint64_t seed) {
    ModelConfig c;
    c.num_layers = dims[0];
    c.num_heads = dims[1];
    c.head_dim = dims[2];
    c.vocab_size = dims[3];
    c.max_positions = dims[4];
    c.init_seed = seed;
    return c;
}

std::vector<const std::vector<float>*> tensors_of(const Model& m) {
    std::vector<const std::vector<float>*> out{&m.token_embedding(), &m.position_embedding()};
    for (int l = 0; l < m.config().num_layers; ++l) {
        const LayerWeights& lw = m.layer(l);
        for (const std::vector<float>* t :
             {&lw.ln1_gain, &lw.ln1_bias, &lw.wq, &lw.bq, &lw.wk, &lw.bk, &lw.wv, &lw.bv,
              &lw.wo, &lw.bo, &lw.ln2_gain, &lw.ln2_bias, &lw.w_fc, &lw.b_fc, &lw.w_proj,
              &lw.b_proj}) {
            out.push_back(t);
        }
    }
    out.push_back(&m.final_ln_gain());
    out.push_back(&m.final_ln_bias());
    out.push_back(&m.lm_head());
    return out;
}

void copy_rows(const std::vector<LogitsRow>& rows, float* out) {
    if (out == nullptr) return;
    size_t at = 0;
    for (const LogitsRow& r : rows) {
        std::memcpy(out + at, r.data(), r.size() * sizeof(float));
        at += r.size();
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- model ---------------------------------------------------------------
int ref_model_init(const int32_t* dims, uint64_t seed, void** out) {
    return guarded([&] { *out = new Model(Model::init(make_cfg(dims, seed))); });
}
int ref_model_load(const char* path, void** out) {
    return guarded([&] { *out = new Model(Model::load(path)); });
}
int ref_model_save(void* m, const char* path) {
    return guarded([&] { static_cast<Model*>(m)->save(path); });
}
void ref_model_free(void* m) { delete static_cast<Model*>(m); }
uint64_t ref_model_checksum(void* m) { return static_cast<Model*>(m)->weight_checksum(); }
int ref_model_tensor_count(void* m) {
    return static_cast<int>(tensors_of(*static_cast<Model*>(m)).size());
}
int ref_model_tensor(void* m, int idx, const float** ptr, int64_t* n) {
    return guarded([&] {
        auto ts = tensors_of(*static_cast<Model*>(m));
        SPECDEC_CHECK(idx >= 0 && idx < static_cast<int>(ts.size()), ContractError,
                      "tensor index out of range");
        *ptr = ts[idx]->data();
        *n = static_cast<int64_t>(ts[idx]->size());
    });
}
int ref_config_validate(const int32_t* dims) {
    return guarded([&] { make_cfg(dims, 0).validate(); });
}

// ---- caches --------------------------------------------------------------
// layout 0 = UnpadArena, 1 = PaddedGrid
int ref_cache_new(int layout, int layers, int batch, int capacity, int kv_dim, void** out) {
    return guarded([&] {
        if (layout == 0) {
            *out = static_cast<CacheArena*>(new UnpadArena(layers, batch, capacity, kv_dim));
        } else {
            *out = static_cast<CacheArena*>(new PaddedGrid(layers, batch, capacity, kv_dim));
        }
    });
}
void ref_cache_free(void* c) { delete static_cast<CacheArena*>(c); }
int ref_cache_committed(void* c, int s, int32_t* out) {
    return guarded([&] { *out = static_cast<CacheArena*>(c)->committed_len(s); });
}
int ref_cache_logical(void* c, int s, int32_t* out) {
    return guarded([&] { *out = static_cast<CacheArena*>(c)->logical_len(s); });
}
int ref_cache_start_offset(void* c, int s, int32_t* out) {
    return guarded([&] {
        auto* u = dynamic_cast<UnpadArena*>(static_cast<CacheArena*>(c));
        SPECDEC_CHECK(u != nullptr, ContractError, "not an unpad arena");
        *out = u->start_offset(s);
    });
}
int ref_cache_commit(void* c, int s, int tau) {
    return guarded([&] {
        auto* u = dynamic_cast<UnpadArena*>(static_cast<CacheArena*>(c));
        SPECDEC_CHECK(u != nullptr, ContractError, "not an unpad arena");
        u->commit_accepted(s, tau);
    });
}
int ref_cache_commit_padded(void* c, const int32_t* samples, const int32_t* taus, int n) {
    return guarded([&] {
        auto* g = dynamic_cast<PaddedGrid*>(static_cast<CacheArena*>(c));
        SPECDEC_CHECK(g != nullptr, ContractError, "not a padded grid");
        g->commit_padded(std::vector<int>(samples, samples + n), std::vector<int>(taus, taus + n));
    });
}
int ref_cache_commit_prefill(void* c, const int32_t* samples, const int32_t* lens, int n) {
    return guarded([&] {
        auto* g = dynamic_cast<PaddedGrid*>(static_cast<CacheArena*>(c));
        SPECDEC_CHECK(g != nullptr, ContractError, "not a padded grid");
        g->commit_prefill(std::vector<int>(samples, samples + n), std::vector<int>(lens, lens + n));
    });
}
int ref_cache_mark_hole(void* c, int s, int pos) {
    return guarded([&] { static_cast<CacheArena*>(c)->mark_hole(s, pos); });
}
int ref_cache_write_kv(void* c, int s, int pos, int layer, const float* k, const float* v) {
    return guarded([&] { static_cast<CacheArena*>(c)->write_kv(s, pos, layer, k, v); });
}
int ref_cache_gather(void* c, int s, int upto, int layer, float* k, float* v, int32_t* count) {
    return guarded(
        [&] { *count = static_cast<CacheArena*>(c)->gather_visible(s, upto, layer, k, v); });
}
int ref_cache_is_pad(void* c, int s, int row, int32_t* out) {
    return guarded([&] {
        auto* g = dynamic_cast<PaddedGrid*>(static_cast<CacheArena*>(c));
        SPECDEC_CHECK(g != nullptr, ContractError, "not a padded grid");
        *out = g->is_pad(s, row) ? 1 : 0;
    });
}
int64_t ref_ledger_useful(void* c) { return static_cast<CacheArena*>(c)->ledger().useful_total(); }
int64_t ref_ledger_padding(void* c) {
    return static_cast<CacheArena*>(c)->ledger().padding_total();
}
int ref_ledger_begin(void* c) {
    return guarded([&] { static_cast<CacheArena*>(c)->ledger().begin_step(); });
}
int ref_ledger_note_tau(void* c, int tau) {
    return guarded([&] { static_cast<CacheArena*>(c)->ledger().note_tau(tau); });
}
int ref_ledger_end(void* c) {
    return guarded([&] { static_cast<CacheArena*>(c)->ledger().end_step(); });
}
int ref_padding_ratio(void* c, double* out) {
    return guarded([&] { *out = padding_ratio(static_cast<CacheArena*>(c)->ledger()); });
}

// ---- ragged --------------------------------------------------------------
int ref_restore_indices(const int32_t* counts, int batch, int flat, int32_t* sample,
                        int32_t* pos) {
    return guarded([&] {
        TokenSlot s = ragged::restore_indices(std::vector<int>(counts, counts + batch), flat);
        *sample = s.original_batch_index;
        *pos = s.original_sequence_position;
    });
}

// ---- forward -------------------------------------------------------------
// Model::forward (model.hpp:71-72): ragged batch + slots with absolute positions.
int ref_forward(void* m, void* c, const int32_t* tokens, const int32_t* counts, int batch,
                const int32_t* slot_sample, const int32_t* slot_pos, float* logits) {
    return guarded([&] {
        std::vector<TokenSequence> per(batch);
        int at = 0;
        for (int s = 0; s < batch; ++s) {
            per[s].assign(tokens + at, tokens + at + counts[s]);
            at += counts[s];
        }
        RaggedBatch rb = ragged::concatenate_inputs(per);
        std::vector<TokenSlot> slots(at);
        for (int i = 0; i < at; ++i) slots[i] = TokenSlot{slot_sample[i], slot_pos[i]};
        copy_rows(static_cast<Model*>(m)->forward(rb, *static_cast<CacheArena*>(c), slots),
                  logits);
    });
}
// Model::forward_planned (model.hpp:76-78).
int ref_forward_planned(void* m, void* c, const int32_t* tokens, int n, const int32_t* sample,
                        const int32_t* logical, const int32_t* slot, const int32_t* store,
                        float* logits) {
    return guarded([&] {
        std::vector<TokenPlan> plans(n);
        for (int i = 0; i < n; ++i) plans[i] = TokenPlan{sample[i], logical[i], slot[i], store[i] != 0};
        copy_rows(static_cast<Model*>(m)->forward_planned(
                      std::vector<TokenId>(tokens, tokens + n), plans,
                      *static_cast<CacheArena*>(c)),
                  logits);
    });
}
int ref_naive_forward(void* m, const int32_t* tokens, int n, float* logits) {
    return guarded([&] {
        copy_rows(testsupport::naive_forward(*static_cast<Model*>(m),
                                             TokenSequence(tokens, tokens + n)),
                  logits);
    });
}

// ---- verify / predictors -------------------------------------------------
int ref_greedy_next(const float* row, int vocab, int32_t* out) {
    return guarded([&] { *out = greedy_next(LogitsRow(row, row + vocab)); });
}
int ref_verify(const float* rows, int nrows, int vocab, const int32_t* drafts, int k,
               int32_t* accepted, int32_t* tau) {
    return guarded([&] {
        std::vector<LogitsRow> rs(nrows);
        for (int i = 0; i < nrows; ++i) rs[i].assign(rows + (size_t)i * vocab, rows + (size_t)(i + 1) * vocab);
        VerifyResult v = verify(rs, TokenSequence(drafts, drafts + k));
        *tau = v.tau;
        for (size_t i = 0; i < v.accepted.size(); ++i) accepted[i] = v.accepted[i];
    });
}
int ref_retrieval_predict(const int32_t* ctx, int n, int match_len, int copy_len, int32_t* out,
                          int32_t* nout) {
    return guarded([&] {
        TokenSequence d = retrieval_predict(TokenSequence(ctx, ctx + n), match_len, copy_len);
        *nout = static_cast<int32_t>(d.size());
        for (size_t i = 0; i < d.size(); ++i) out[i] = d[i];
    });
}
int ref_synthetic_predict(const int32_t* ctx, int n, int k, void* target, double acc,
                          uint64_t step_seed, int32_t* out) {
    return guarded([&] {
        TokenSequence d = synthetic_predict(TokenSequence(ctx, ctx + n), k,
                                            *static_cast<Model*>(target), acc, step_seed);
        for (size_t i = 0; i < d.size(); ++i) out[i] = d[i];
    });
}
uint64_t ref_mix_seed(uint64_t a, uint64_t b, uint64_t c) { return mix_seed(a, b, c); }

// ---- engine --------------------------------------------------------------
// mode: 0 greedy, 1 vanilla, 2 ems; predictor: 0 draft, 1 retrieval, 2 synthetic.
// Writes results_json (engine.cpp:531-587) into json_out (truncated to cap).
int ref_decode(int mode, int predictor, int k, int match_len, int copy_len, int batch,
               int max_new, int stop_on_eos, uint64_t seed, double accuracy, void* target,
               void* draft, const char* const* prompts, char* json_out, int64_t cap,
               int64_t* json_len) {
    return guarded([&] {
        EngineConfig cfg;
        cfg.mode = static_cast<Mode>(mode);
        cfg.predictor = static_cast<PredictorKind>(predictor);
        cfg.k = k;
        cfg.match_len = match_len;
        cfg.copy_len = copy_len;
        cfg.batch_size = batch;
        cfg.max_new_tokens = max_new;
        cfg.stop_on_eos = stop_on_eos != 0;
        cfg.seed = seed;
        cfg.synthetic_accuracy = accuracy;
        std::vector<std::string> ps(prompts, prompts + batch);
        DecodeResult r = cfg.mode == Mode::greedy
                             ? decode_greedy(ps, cfg, *static_cast<Model*>(target))
                             : decode_speculative(ps, cfg, *static_cast<Model*>(target),
                                                  static_cast<Model*>(draft));
        std::string js = results_json(cfg, r);
        *json_len = static_cast<int64_t>(js.size());
        if (json_out != nullptr && cap > 0) {
            size_t n = std::min<size_t>(js.size(), static_cast<size_t>(cap - 1));
            std::memcpy(json_out, js.data(), n);
            json_out[n] = 0;
        }
    });
}

}  // extern "C"
