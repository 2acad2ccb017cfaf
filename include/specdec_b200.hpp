// C++ layer over the C ABI: the reference's hot-path types
// and calls re-exposed on the B200 library, with the reference's names,
// argument meaning and exception types, so code written against
// /root/reference/proj/include/specdec/{common,ragged,model,kv_cache,engine}.hpp
// recompiles against this header and links libspecdec_b200.so.
//
//   specdec::Error / ConfigError / CapacityError / ContractError / IoError  common.hpp:13-34
//   specdec::RaggedBatch, TokenSlot, ragged::concatenate_inputs,
//     ragged::restore_indices, ragged::attention_extent                      ragged.hpp:13-45
//   specdec::ModelConfig, TokenPlan, greedy_next, Model                       model.hpp:14-103
//   specdec::CacheArena, UnpadArena, PaddedGrid                               kv_cache.hpp:68-168
//   specdec::VerifyResult, verify                                             engine.hpp:82-90
//   specdec::draft_predict, retrieval_predict, synthetic_predict              predictors.hpp:13-20
//   specdec::Mode, PredictorKind, EngineConfig, SampleStep, StepRecord,
//     RunMetrics, DecodeResult, make_step_record, compute_metrics,
//     decode_greedy, decode_speculative, results_json                         engine.hpp:15-110
//
//   specdec::LedgerStep, WriteLedger, padding_ratio                           kv_cache.hpp:13-62
//   specdec::softmax, LayerWeights, Model weight accessors                     model.hpp:27-32, 48, 81-87
//   specdec::SplitMix64, mix_seed                                              rng.hpp
//   specdec::tok::tokenize / detokenize                                        tokenizer.hpp
//
// Differences, all at the boundary: a Model lives on one GPU (precision
// SD_FP32_CHECK -- bit-exact with the reference -- unless SD_BF16 is asked
// for); a cache arena is a device arena on device 0 from construction (fp32),
// and the first Model that runs a forward over it binds it (same depth and
// width; the arena then takes the model's head split, precision and device,
// which needs it to be still unwritten if they differ).  Weight accessors
// download the tensors on first use (bf16 models return their bf16 values
// widened to fp32).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "specdec_b200.h"

namespace specdec {

using TokenId = int32_t;
using TokenSequence = std::vector<TokenId>;
using LogitsRow = std::vector<float>;

// ------------------------------------------------------------ SplitMix64 (rng.hpp)
class SplitMix64 {
public:
    explicit SplitMix64(uint64_t seed) : state_(seed) {}
    uint64_t next_u64() {
        uint64_t z = (state_ += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    float next_unit_float() { return static_cast<float>(next_u64() >> 40) * 0x1.0p-24f; }
    double next_unit_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    float next_symmetric(float limit) { return (2.0f * next_unit_float() - 1.0f) * limit; }

private:
    uint64_t state_;
};
inline uint64_t mix_seed(uint64_t a, uint64_t b = 0, uint64_t c = 0) {
    SplitMix64 r(a ^ (b * 0xD1B54A32D192ED03ULL) ^ (c * 0x8CB92BA72F3D8DD7ULL));
    return r.next_u64();
}

// ------------------------------------------------------------ errors (common.hpp:13-34)
struct Error : std::runtime_error {
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
struct ConfigError : Error {
    explicit ConfigError(const std::string& msg) : Error("config: " + msg) {}
};
struct CapacityError : Error {
    explicit CapacityError(const std::string& msg) : Error("capacity: " + msg) {}
};
struct ContractError : Error {
    explicit ContractError(const std::string& msg) : Error("contract: " + msg) {}
};
struct IoError : Error {
    explicit IoError(const std::string& msg) : Error("io: " + msg) {}
};

namespace b200 {
// Rethrow a C-ABI status as the reference's exception type (the library's
// message already carries the reference's "config: " / ... prefix).
inline void check(int rc) {
    if (rc == SD_OK) return;
    std::string m = sd_last_error();
    auto strip = [&](const char* p) {
        const std::string s(p);
        return m.compare(0, s.size(), s) == 0 ? m.substr(s.size()) : m;
    };
    switch (rc) {
        case SD_CONFIG: throw ConfigError(strip("config: "));
        case SD_CAPACITY: throw CapacityError(strip("capacity: "));
        case SD_CONTRACT: throw ContractError(strip("contract: "));
        case SD_IO: throw IoError(strip("io: "));
        default: throw Error(m);
    }
}
}  // namespace b200

// ------------------------------------------------------------ byte tokenizer (tokenizer.hpp)
namespace tok {
constexpr TokenId kBos = 0;
constexpr TokenId kEos = 1;
constexpr TokenId kPad = 2;
constexpr TokenId kByteOffset = 3;
constexpr int kVocabSize = 259;
inline TokenSequence tokenize(const std::string& text) {
    TokenSequence out;
    for (unsigned char ch : text) out.push_back(static_cast<TokenId>(ch) + kByteOffset);
    return out;
}
inline std::string detokenize(const TokenSequence& tokens) {
    std::string out;
    for (TokenId id : tokens) {
        if (id < 0 || id >= kVocabSize) throw ContractError("token id " + std::to_string(id) + " outside vocabulary");
        if (id < kByteOffset) throw ContractError("special token " + std::to_string(id) + " has no byte form");
        out.push_back(static_cast<char>(id - kByteOffset));
    }
    return out;
}
inline bool is_special(TokenId id) { return id >= 0 && id < kByteOffset; }
}  // namespace tok

// ------------------------------------------------------------ ragged batching (ragged.hpp)
struct RaggedBatch {
    std::vector<TokenId> concatenated_tokens;
    std::vector<int> token_nums_per_sample;
    int total_input_token_nums = 0;
    int batch_size() const { return static_cast<int>(token_nums_per_sample.size()); }
};

struct TokenSlot {
    int original_batch_index = 0;
    int original_sequence_position = 0;
    bool operator==(const TokenSlot&) const = default;
};

namespace ragged {
// Algorithm 1 (ragged.cpp:6-17): flatten in order, zero-length samples keep their entry.
inline RaggedBatch concatenate_inputs(const std::vector<TokenSequence>& per_sample) {
    if (per_sample.empty()) throw ContractError("batch must have at least one sample");
    RaggedBatch b;
    for (const TokenSequence& s : per_sample) {
        b.concatenated_tokens.insert(b.concatenated_tokens.end(), s.begin(), s.end());
        b.token_nums_per_sample.push_back(static_cast<int>(s.size()));
        b.total_input_token_nums += static_cast<int>(s.size());
    }
    return b;
}
// Algorithm 2 (ragged.cpp:19-36), through the library (ContractError out of range).
inline TokenSlot restore_indices(const std::vector<int>& counts, int flat_index) {
    std::vector<int32_t> c(counts.begin(), counts.end());
    int32_t s = 0, p = 0;
    b200::check(sd_restore_indices(c.data(), static_cast<int>(c.size()), flat_index, &s, &p));
    return TokenSlot{s, p};
}
inline int attention_extent(const TokenSlot& slot, int cache_committed_len) {
    return cache_committed_len + slot.original_sequence_position + 1;
}
}  // namespace ragged

// ------------------------------------------------------------ model (model.hpp)
struct ModelConfig {
    int num_layers = 2;
    int num_heads = 2;
    int head_dim = 16;
    int vocab_size = tok::kVocabSize;
    int max_positions = 512;
    uint64_t init_seed = 0xD5EED;

    int hidden() const { return num_heads * head_dim; }
    int mlp_hidden() const { return 4 * hidden(); }
    sd_model_config c() const {
        return sd_model_config{num_layers, num_heads, head_dim, vocab_size, max_positions, init_seed};
    }
    void validate() const {
        const sd_model_config cfg = c();
        b200::check(sd_config_validate(&cfg));
    }
};

struct TokenPlan {
    int sample = 0;
    int logical_pos = 0;
    int write_slot = 0;
    bool store = true;
};

// Numerically safe softmax (model.cpp:20-32), host-side helper of the tests.
inline std::vector<float> softmax(const std::vector<float>& scores) {
    if (scores.empty()) throw ContractError("softmax over an empty set");
    float mx = scores[0];
    for (float v : scores) mx = std::max(mx, v);
    std::vector<float> out(scores.size());
    float denom = 0.0f;
    for (size_t i = 0; i < scores.size(); ++i) {
        out[i] = std::exp(scores[i] - mx);
        denom += out[i];
    }
    for (float& w : out) w /= denom;
    return out;
}

// Argmax with ties toward the lowest id (model.cpp:34-41).
inline TokenId greedy_next(const LogitsRow& row) {
    if (row.empty()) throw ContractError("argmax over an empty row");
    TokenId best = 0;
    for (size_t i = 1; i < row.size(); ++i)
        if (row[i] > row[best]) best = static_cast<TokenId>(i);
    return best;
}

// ------------------------------------------------------------ write ledger (kv_cache.hpp:13-62)
struct LedgerStep {
    std::vector<int> tau_list;
    int tau_max = 0;
    int64_t pad_writes = 0;
    int64_t useful_writes = 0;
};

// A standalone WriteLedger(batch) owns its library ledger; a cache's ledger()
// is a view of the ledger the library keeps for that cache.
class WriteLedger {
public:
    explicit WriteLedger(int batch_size) {
        sd_ledger* l = nullptr;
        b200::check(sd_ledger_create(batch_size, &l));
        h_.reset(l, sd_ledger_destroy);
    }
    explicit WriteLedger(sd_ledger* view) : h_(view, [](sd_ledger*) {}) {}

    void note_useful(int sample) { b200::check(sd_ledger_note_useful(h_.get(), sample)); }
    void note_padding(int sample) { b200::check(sd_ledger_note_padding(h_.get(), sample)); }
    void begin_step() { b200::check(sd_ledger_begin_step(h_.get())); }
    void note_tau(int tau) { b200::check(sd_ledger_note_tau(h_.get(), tau)); }
    void end_step() { b200::check(sd_ledger_end_step(h_.get())); }

    int64_t useful_total() const { return totals().first; }
    int64_t padding_total() const { return totals().second; }
    int64_t total() const { return useful_total() + padding_total(); }
    const std::vector<int64_t>& useful_by_sample() const {
        by_sample();
        return useful_by_;
    }
    const std::vector<int64_t>& padding_by_sample() const {
        by_sample();
        return padding_by_;
    }
    const std::vector<LedgerStep>& steps() const {
        int64_t n = 0;
        b200::check(sd_ledger_num_steps(h_.get(), &n));
        steps_.assign(static_cast<size_t>(n), LedgerStep{});
        for (int64_t i = 0; i < n; ++i) {
            LedgerStep& st = steps_[static_cast<size_t>(i)];
            int32_t nt = 0, tm = 0;
            std::vector<int32_t> buf(64);
            b200::check(sd_ledger_step(h_.get(), i, buf.data(), 64, &nt, &tm, &st.pad_writes, &st.useful_writes));
            if (nt > 64) {
                buf.resize(static_cast<size_t>(nt));
                b200::check(sd_ledger_step(h_.get(), i, buf.data(), nt, &nt, &tm, &st.pad_writes, &st.useful_writes));
            }
            st.tau_list.assign(buf.begin(), buf.begin() + nt);
            st.tau_max = tm;
        }
        return steps_;
    }
    std::string dump_json() const {
        int64_t n = 0;
        b200::check(sd_ledger_dump_json(h_.get(), nullptr, 0, &n));
        std::string out(static_cast<size_t>(n) + 1, '\0');
        b200::check(sd_ledger_dump_json(h_.get(), out.data(), n + 1, &n));
        out.resize(static_cast<size_t>(n));
        return out;
    }
    const sd_ledger* handle() const { return h_.get(); }

private:
    std::pair<int64_t, int64_t> totals() const {
        int64_t u = 0, p = 0;
        b200::check(sd_ledger_totals(h_.get(), &u, &p));
        return {u, p};
    }
    void by_sample() const {
        int32_t b = 0;
        b200::check(sd_ledger_batch(h_.get(), &b));
        useful_by_.assign(static_cast<size_t>(b), 0);
        padding_by_.assign(static_cast<size_t>(b), 0);
        b200::check(sd_ledger_by_sample(h_.get(), useful_by_.data(), padding_by_.data()));
    }
    std::shared_ptr<sd_ledger> h_;
    mutable std::vector<int64_t> useful_by_, padding_by_;
    mutable std::vector<LedgerStep> steps_;
};

// padding_ratio (kv_cache.cpp:64-76); ContractError without steps.
inline double padding_ratio(const WriteLedger& ledger) {
    double r = 0.0;
    b200::check(sd_ledger_padding_ratio(ledger.handle(), &r));
    return r;
}

// ------------------------------------------------------------ KV arenas (kv_cache.hpp:65-168)
// Read contract shared by both layouts.  The device arena exists from
// construction; the first Model::forward over it binds the model.
class CacheArena {
public:
    CacheArena(int num_layers, int batch_size, int capacity, int kv_dim, int layout)
        : num_layers_(num_layers), batch_size_(batch_size), capacity_(capacity), kv_dim_(kv_dim) {
        sd_cache* c = nullptr;
        b200::check(sd_cache_create_dims(num_layers, batch_size, capacity, kv_dim, layout, 0, SD_FP32_CHECK, &c));
        h_.reset(c, sd_cache_destroy);
        sd_ledger* l = nullptr;
        b200::check(sd_cache_ledger_handle(c, &l));
        ledger_ = std::make_unique<WriteLedger>(l);
    }
    virtual ~CacheArena() = default;
    CacheArena(const CacheArena&) = delete;
    CacheArena& operator=(const CacheArena&) = delete;

    int num_layers() const { return num_layers_; }
    int batch_size() const { return batch_size_; }
    int capacity() const { return capacity_; }
    int kv_dim() const { return kv_dim_; }

    int committed_len(int sample) const {
        int32_t v = 0;
        b200::check(sd_cache_committed_len(h_.get(), sample, &v));
        return v;
    }
    int logical_len(int sample) const {
        int32_t v = 0;
        b200::check(sd_cache_logical_len(h_.get(), sample, &v));
        return v;
    }
    // Store a real token's key/value for one layer; counted once, on layer 0.
    void write_kv(int sample, int position, int layer, const float* k_vec, const float* v_vec) {
        b200::check(sd_cache_write_kv(h_.get(), sample, position, layer, k_vec, v_vec));
    }
    virtual void mark_hole(int sample, int position) { b200::check(sd_cache_mark_hole(h_.get(), sample, position)); }
    // Copies the visible real K/V rows [0, upto] of (sample, layer), ascending.
    int gather_visible(int sample, int upto, int layer, float* k_out, float* v_out) const {
        int32_t n = 0;
        b200::check(sd_cache_gather_visible(h_.get(), sample, upto, layer, k_out, v_out, &n));
        return n;
    }
    const WriteLedger& ledger() const { return *ledger_; }
    WriteLedger& ledger() { return *ledger_; }

    sd_cache* handle() const { return h_.get(); }

protected:
    int num_layers_, batch_size_, capacity_, kv_dim_;
    std::shared_ptr<sd_cache> h_;
    std::unique_ptr<WriteLedger> ledger_;
};

// EMS-SD layout (kv_cache.hpp:105-128).
class UnpadArena : public CacheArena {
public:
    UnpadArena(int num_layers, int batch_size, int capacity, int kv_dim)
        : CacheArena(num_layers, batch_size, capacity, kv_dim, SD_UNPAD) {}
    int start_offset(int sample) const {
        int32_t v = 0;
        b200::check(sd_cache_start_offset(h_.get(), sample, &v));
        return v;
    }
    void commit_accepted(int sample, int tau) { b200::check(sd_cache_commit_accepted(h_.get(), sample, tau)); }
};

// Vanilla (aligned) layout (kv_cache.hpp:133-168).
class PaddedGrid : public CacheArena {
public:
    PaddedGrid(int num_layers, int batch_size, int capacity, int kv_dim)
        : CacheArena(num_layers, batch_size, capacity, kv_dim, SD_PADDED) {}
    bool is_pad(int sample, int row) const {
        int32_t v = 0;
        b200::check(sd_cache_is_pad(h_.get(), sample, row, &v));
        return v != 0;
    }
    void commit_prefill(const std::vector<int>& samples, const std::vector<int>& prompt_lens) {
        if (samples.size() != prompt_lens.size()) throw ContractError("commit_prefill: mismatched lists");
        std::vector<int32_t> s(samples.begin(), samples.end()), l(prompt_lens.begin(), prompt_lens.end());
        b200::check(sd_cache_commit_prefill(h_.get(), s.data(), l.data(), static_cast<int>(s.size())));
    }
    void commit_padded(const std::vector<int>& samples, const std::vector<int>& taus) {
        if (samples.empty() || samples.size() != taus.size())
            throw ContractError("padded commit needs matching sample and tau lists");
        std::vector<int32_t> s(samples.begin(), samples.end()), t(taus.begin(), taus.end());
        b200::check(sd_cache_commit_padded(h_.get(), s.data(), t.data(), static_cast<int>(s.size())));
    }
};

// One layer's tensors (model.hpp:27-32), declaration order.
struct LayerWeights {
    std::vector<float> ln1_gain, ln1_bias;
    std::vector<float> wq, bq, wk, bk, wv, bv, wo, bo;
    std::vector<float> ln2_gain, ln2_bias;
    std::vector<float> w_fc, b_fc, w_proj, b_proj;
};

// Decoder-only transformer resident on one B200 (model.hpp:54-103).
class Model {
public:
    static Model init(const ModelConfig& config, int precision = SD_FP32_CHECK, int device = 0) {
        config.validate();
        const sd_model_config c = config.c();
        sd_model* m = nullptr;
        b200::check(sd_model_init(&c, device, precision, &m));
        return Model(m, config);
    }
    static Model load(const std::string& path, int precision = SD_FP32_CHECK, int device = 0) {
        sd_model* m = nullptr;
        b200::check(sd_model_load(path.c_str(), device, precision, &m));
        sd_model_config c{};
        b200::check(sd_model_get_config(m, &c));
        return Model(m, ModelConfig{c.num_layers, c.num_heads, c.head_dim, c.vocab_size, c.max_positions,
                                    c.init_seed});
    }
    void save(const std::string& path) const { b200::check(sd_model_save(h_.get(), path.c_str())); }

    const ModelConfig& config() const { return config_; }
    uint64_t weight_checksum() const {
        uint64_t v = 0;
        b200::check(sd_model_checksum(h_.get(), &v));
        return v;
    }

    // Ragged entry point (model.cpp:235-254): slot i must be
    // restore_indices(batch.token_nums_per_sample, i) at the sample's committed extent.
    std::vector<LogitsRow> forward(const RaggedBatch& batch, CacheArena& cache,
                                   const std::vector<TokenSlot>& slots) const {
        const int T = batch.total_input_token_nums;
        if (static_cast<int>(slots.size()) != T || static_cast<int>(batch.concatenated_tokens.size()) != T)
            throw ContractError("forward: slots / tokens do not match the batch");
        std::vector<int32_t> counts(batch.token_nums_per_sample.begin(), batch.token_nums_per_sample.end());
        std::vector<int32_t> ss(T), sp(T);
        for (int i = 0; i < T; ++i) {
            ss[i] = slots[i].original_batch_index;
            sp[i] = slots[i].original_sequence_position;
        }
        std::vector<float> flat(static_cast<size_t>(T) * config_.vocab_size);
        b200::check(sd_forward(h_.get(), cache.handle(), batch.concatenated_tokens.data(), counts.data(),
                               batch.batch_size(), ss.data(), sp.data(), flat.data(), nullptr));
        return rows(flat, T);
    }

    // Plan-level entry point (model.cpp:256-373).
    std::vector<LogitsRow> forward_planned(const std::vector<TokenId>& tokens, const std::vector<TokenPlan>& plans,
                                           CacheArena& cache) const {
        const int T = static_cast<int>(tokens.size());
        if (static_cast<int>(plans.size()) != T) throw ContractError("forward_planned: tokens / plans mismatch");
        std::vector<int32_t> s(T), lp(T), ws(T), st(T);
        for (int i = 0; i < T; ++i) {
            s[i] = plans[i].sample;
            lp[i] = plans[i].logical_pos;
            ws[i] = plans[i].write_slot;
            st[i] = plans[i].store ? 1 : 0;
        }
        std::vector<float> flat(static_cast<size_t>(T) * config_.vocab_size);
        b200::check(sd_forward_planned(h_.get(), cache.handle(), tokens.data(), T, s.data(), lp.data(), ws.data(),
                                       st.data(), flat.data(), nullptr));
        return rows(flat, T);
    }

    // Weight access for independent reimplementations in tests (model.hpp:81-87).
    const std::vector<float>& token_embedding() const { return tensor(-1, 0); }
    const std::vector<float>& position_embedding() const { return tensor(-1, 1); }
    const std::vector<float>& final_ln_gain() const { return tensor(-1, 2); }
    const std::vector<float>& final_ln_bias() const { return tensor(-1, 3); }
    const std::vector<float>& lm_head() const { return tensor(-1, 4); }
    const LayerWeights& layer(int i) const {
        if (i < 0 || i >= config_.num_layers) throw std::out_of_range("layer index out of range");
        auto& lw = weights_->layers;
        if (lw.empty()) lw.resize(static_cast<size_t>(config_.num_layers));
        LayerWeights& w = lw[static_cast<size_t>(i)];
        if (w.ln1_gain.empty()) {
            std::vector<float>* t[16] = {&w.ln1_gain, &w.ln1_bias, &w.wq, &w.bq, &w.wk, &w.bk, &w.wv, &w.bv,
                                         &w.wo, &w.bo, &w.ln2_gain, &w.ln2_bias, &w.w_fc, &w.b_fc, &w.w_proj,
                                         &w.b_proj};
            for (int k = 0; k < 16; ++k) fetch(i, k, *t[k]);
        }
        return w;
    }

    sd_model* handle() const { return h_.get(); }

private:
    struct Weights {
        std::vector<float> model_level[5];
        std::vector<LayerWeights> layers;
    };
    Model(sd_model* m, const ModelConfig& c) : h_(m, sd_model_destroy), config_(c), weights_(std::make_shared<Weights>()) {}
    std::vector<LogitsRow> rows(const std::vector<float>& flat, int T) const {
        std::vector<LogitsRow> out(T);
        for (int i = 0; i < T; ++i)
            out[i].assign(flat.begin() + static_cast<size_t>(i) * config_.vocab_size,
                          flat.begin() + static_cast<size_t>(i + 1) * config_.vocab_size);
        return out;
    }
    int64_t tensor_size(int layer, int k) const {
        const int64_t h = config_.hidden(), m = config_.mlp_hidden(), V = config_.vocab_size,
                      P = config_.max_positions;
        if (layer < 0) {
            const int64_t sz[5] = {V * h, P * h, h, h, V * h};
            return sz[k];
        }
        const int64_t sz[16] = {h, h, h * h, h, h * h, h, h * h, h, h * h, h, h, h, m * h, m, h * m, h};
        return sz[k];
    }
    void fetch(int layer, int k, std::vector<float>& out) const {
        out.resize(static_cast<size_t>(tensor_size(layer, k)));
        b200::check(sd_model_get_tensor(h_.get(), layer, k, out.data(), static_cast<int64_t>(out.size())));
    }
    const std::vector<float>& tensor(int layer, int k) const {
        std::vector<float>& t = weights_->model_level[k];
        if (t.empty()) fetch(layer, k, t);
        return t;
    }
    std::shared_ptr<sd_model> h_;
    ModelConfig config_;
    std::shared_ptr<Weights> weights_;  // lazily downloaded copies
};

// ------------------------------------------------------------ verify (engine.hpp:82-90)
struct VerifyResult {
    TokenSequence accepted;
    int tau = 0;
};

// engine.cpp:60-76: accept the longest prefix of drafts that the target's
// greedy picks reproduce, then the target's own token at the first mismatch
// (or the bonus token after all of them).
inline VerifyResult verify(const std::vector<LogitsRow>& rows, const TokenSequence& drafts) {
    if (rows.size() != drafts.size() + 1) throw ContractError("verify needs one more row than drafts");
    VerifyResult r;
    for (size_t j = 0; j < rows.size(); ++j) {
        const TokenId x = greedy_next(rows[j]);
        r.accepted.push_back(x);
        if (j == drafts.size() || x != drafts[j]) break;
    }
    r.tau = static_cast<int>(r.accepted.size());
    return r;
}

// ------------------------------------------------------------ predictors (predictors.hpp:13-20)
// Draft / synthetic rollouts run on the GPU through the given Model.
inline TokenSequence draft_predict(const TokenSequence& context, int k, const Model& draft) {
    TokenSequence out(static_cast<size_t>(std::max(k, 0)));
    b200::check(sd_draft_predict(draft.handle(), context.data(), static_cast<int>(context.size()), k, out.data()));
    return out;
}
inline TokenSequence retrieval_predict(const TokenSequence& context, int match_len, int copy_len) {
    TokenSequence out(static_cast<size_t>(std::max(copy_len, 0)));
    int32_t n = 0;
    b200::check(sd_retrieval_predict(context.data(), static_cast<int>(context.size()), match_len, copy_len, out.data(),
                                     &n));
    out.resize(static_cast<size_t>(n));
    return out;
}
inline TokenSequence synthetic_predict(const TokenSequence& context, int k, const Model& target, double accuracy,
                                       uint64_t step_seed) {
    TokenSequence out(static_cast<size_t>(std::max(k, 0)));
    b200::check(sd_synthetic_predict(target.handle(), context.data(), static_cast<int>(context.size()), k, accuracy,
                                     step_seed, out.data()));
    return out;
}

// ------------------------------------------------------------ engine (engine.hpp:15-110)
// The reference's decoding entry points over sd_decode (the library's engine:
// prefill, then the verify-step loop of engine.cpp:391-489 with the
// predictors on the host, every forward on the GPU), plus the host-side
// bookkeeping of engine.cpp (step records, metrics, the JSON run report).
enum class Mode { greedy, vanilla, ems };
enum class PredictorKind { draft, retrieval, synthetic };

inline Mode mode_from_string(const std::string& name) {
    if (name == "greedy") return Mode::greedy;
    if (name == "vanilla") return Mode::vanilla;
    if (name == "ems") return Mode::ems;
    throw ConfigError("unknown mode '" + name + "' (greedy, vanilla, ems)");
}
inline std::string to_string(Mode mode) {
    return mode == Mode::greedy ? "greedy" : mode == Mode::vanilla ? "vanilla" : "ems";
}
inline PredictorKind predictor_from_string(const std::string& name) {
    if (name == "draft") return PredictorKind::draft;
    if (name == "retrieval") return PredictorKind::retrieval;
    if (name == "synthetic") return PredictorKind::synthetic;
    throw ConfigError("unknown predictor '" + name + "' (draft, retrieval, synthetic)");
}
inline std::string to_string(PredictorKind kind) {
    return kind == PredictorKind::draft ? "draft" : kind == PredictorKind::retrieval ? "retrieval" : "synthetic";
}

struct EngineConfig {
    Mode mode = Mode::ems;
    PredictorKind predictor = PredictorKind::draft;
    int k = 4;
    int match_len = 2;
    int copy_len = 7;
    int batch_size = 1;
    int max_new_tokens = 64;
    bool stop_on_eos = true;
    uint64_t seed = 1;
    double synthetic_accuracy = 0.8;

    // engine.cpp:48-58
    void validate() const {
        if (predictor != PredictorKind::retrieval && k < 1) throw ConfigError("k must be >= 1");
        if (match_len < 1) throw ConfigError("match_len must be >= 1");
        if (copy_len < 1) throw ConfigError("copy_len must be >= 1");
        if (batch_size < 1) throw ConfigError("batch_size must be >= 1");
        if (max_new_tokens < 0) throw ConfigError("max_new_tokens must be >= 0");
        if (!(synthetic_accuracy >= 0.0 && synthetic_accuracy < 1.0))
            throw ConfigError("synthetic accuracy must lie in [0, 1)");
    }
    sd_engine_config c() const {
        sd_engine_config e{};
        e.mode = static_cast<int32_t>(mode);
        e.predictor = static_cast<int32_t>(predictor);
        e.k = k;
        e.match_len = match_len;
        e.copy_len = copy_len;
        e.batch_size = batch_size;
        e.max_new_tokens = max_new_tokens;
        e.stop_on_eos = stop_on_eos ? 1 : 0;
        e.seed = seed;
        e.synthetic_accuracy = synthetic_accuracy;
        e.sample_id_base = 0;
        return e;
    }
};

struct SampleStep {
    int sample = 0;
    int k = 0;
    int input_padding = 0;
    int tau = 0;
    int kv_padding = 0;
    bool clipped = false;
};

struct StepRecord {
    std::vector<SampleStep> samples;
    int tau_max = 0;
    double delta_bar = 0.0;
    double r_bar = 0.0;
};

struct RunMetrics {
    int decode_steps = 0;
    std::vector<int64_t> tokens_generated;
    int64_t total_tokens_generated = 0;
    double avg_acceptance_length = 0.0;
    double avg_padding_ratio = 0.0;
    int64_t total_input_padding = 0;
    int64_t total_kv_padding = 0;
    int64_t useful_kv_writes = 0;
    int64_t padding_kv_writes = 0;
    int64_t real_tokens_processed = 0;
    int64_t pad_tokens_processed = 0;
    int64_t total_tokens_processed = 0;
    double prefill_seconds = 0.0;
    double decode_seconds = 0.0;
    double tokens_per_second_decode = 0.0;
    double tokens_per_second_total = 0.0;
};

struct DecodeResult {
    std::vector<TokenSequence> generated_tokens;
    std::vector<std::string> texts;
    std::vector<StepRecord> steps;
    RunMetrics metrics;
    std::string ledger_json;
};

// engine.cpp:78-105
inline StepRecord make_step_record(const std::vector<int>& sample_ids, const std::vector<int>& ks,
                                   const std::vector<int>& taus, const std::vector<bool>& clipped) {
    const size_t n = sample_ids.size();
    if (n < 1) throw ContractError("a step needs at least one sample");
    if (ks.size() != n || taus.size() != n || clipped.size() != n)
        throw ContractError("per-sample step lists differ in length");
    int k_max = 0, tau_max = 0;
    double tau_sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
        if (ks[i] < 0) throw ContractError("negative draft count");
        if (taus[i] < 1 || taus[i] > ks[i] + 1) throw ContractError("acceptance length outside [1, k + 1]");
        k_max = std::max(k_max, ks[i]);
        tau_max = std::max(tau_max, taus[i]);
        tau_sum += taus[i];
    }
    StepRecord r;
    r.samples.resize(n);
    for (size_t i = 0; i < n; ++i)
        r.samples[i] = SampleStep{sample_ids[i], ks[i], k_max - ks[i], taus[i], tau_max - taus[i], clipped[i]};
    r.tau_max = tau_max;
    r.delta_bar = tau_max - tau_sum / static_cast<double>(n);
    r.r_bar = r.delta_bar / static_cast<double>(tau_max);
    return r;
}

// engine.cpp:107-126
inline RunMetrics compute_metrics(const std::vector<StepRecord>& records) {
    RunMetrics m;
    m.decode_steps = static_cast<int>(records.size());
    if (records.empty()) return m;
    int64_t events = 0;
    double tau_sum = 0.0, ratio_sum = 0.0;
    for (const StepRecord& rec : records) {
        for (const SampleStep& s : rec.samples) {
            tau_sum += s.tau;
            m.total_input_padding += s.input_padding;
            m.total_kv_padding += s.kv_padding;
            ++events;
        }
        ratio_sum += rec.r_bar;
    }
    m.avg_acceptance_length = tau_sum / static_cast<double>(events);
    m.avg_padding_ratio = ratio_sum / static_cast<double>(records.size());
    return m;
}

namespace b200 {
inline std::string text_without_specials(const TokenSequence& tokens) {  // engine.cpp:148-155
    TokenSequence bytes;
    for (TokenId t : tokens)
        if (!tok::is_special(t)) bytes.push_back(t);
    return tok::detokenize(bytes);
}

// sd_decode, then the reference's result assembly (engine.cpp:206-289, 291-528)
inline DecodeResult run_decode(const std::vector<std::string>& prompts, const EngineConfig& config,
                               const Model& target, const Model* draft) {
    const int b = config.batch_size;
    std::vector<int32_t> flat, lens;
    for (const std::string& p : prompts) {  // engine.cpp:136-145: BOS + byte tokens
        flat.push_back(tok::kBos);
        for (TokenId t : tok::tokenize(p)) flat.push_back(t);
        lens.push_back(static_cast<int32_t>(tok::tokenize(p).size() + 1));
    }
    const int mx = std::max(config.max_new_tokens, 1);
    std::vector<int32_t> gen(static_cast<size_t>(b) * mx), cnt(b);
    const int64_t cap = static_cast<int64_t>(b) * (config.max_new_tokens + 2) + 16;
    std::vector<int32_t> rec(static_cast<size_t>(cap) * 6);
    int64_t n_rec = 0, ledger[2] = {0, 0};
    double timing[2] = {0.0, 0.0};
    const sd_engine_config c = config.c();
    check(sd_decode(&c, target.handle(), draft ? draft->handle() : nullptr, flat.data(), lens.data(), gen.data(),
                    cnt.data(), rec.data(), cap, &n_rec, ledger, timing));

    DecodeResult out;
    out.metrics.tokens_generated.assign(b, 0);
    for (int s = 0; s < b; ++s) {
        TokenSequence g(gen.begin() + static_cast<size_t>(s) * mx, gen.begin() + static_cast<size_t>(s) * mx + cnt[s]);
        out.texts.push_back(text_without_specials(g));
        out.generated_tokens.push_back(std::move(g));
        out.metrics.tokens_generated[s] = cnt[s];
        out.metrics.total_tokens_generated += cnt[s];
    }
    RunMetrics& m = out.metrics;
    m.prefill_seconds = timing[0];
    m.decode_seconds = timing[1];
    m.useful_kv_writes = ledger[0];
    m.padding_kv_writes = ledger[1];
    std::string led = "[]";
    if (config.max_new_tokens > 0 && config.mode == Mode::greedy) {  // engine.cpp:259-287
        for (int s = 0; s < b; ++s) {
            m.real_tokens_processed += lens[s] + cnt[s] - 1;
            m.decode_steps = std::max(m.decode_steps, cnt[s] - 1);
        }
        m.avg_acceptance_length = 1.0;
        m.total_tokens_processed = m.real_tokens_processed;
    } else if (config.max_new_tokens > 0) {  // engine.cpp:486-528
        // step records: rows {step, sample, k, tau, clipped, 0}, grouped by step
        for (int64_t i = 0; i < n_rec;) {
            const int step = rec[i * 6];
            std::vector<int> ids, ks, taus;
            std::vector<bool> clips;
            for (; i < n_rec && rec[i * 6] == step; ++i) {
                ids.push_back(rec[i * 6 + 1]);
                ks.push_back(rec[i * 6 + 2]);
                taus.push_back(rec[i * 6 + 3]);
                clips.push_back(rec[i * 6 + 4] != 0);
            }
            out.steps.push_back(make_step_record(ids, ks, taus, clips));
        }
        const RunMetrics agg = compute_metrics(out.steps);
        m.decode_steps = agg.decode_steps;
        m.avg_acceptance_length = agg.avg_acceptance_length;
        m.avg_padding_ratio = agg.avg_padding_ratio;
        m.total_input_padding = agg.total_input_padding;
        m.total_kv_padding = agg.total_kv_padding;
        for (int s = 0; s < b; ++s) m.real_tokens_processed += lens[s];
        led = "[";
        for (size_t i = 0; i < out.steps.size(); ++i) {  // WriteLedger::dump_json (kv_cache.cpp:53-62)
            const StepRecord& r = out.steps[i];
            int64_t pad = 0, useful = 0;
            std::string taus = "[";
            for (size_t j = 0; j < r.samples.size(); ++j) {
                const SampleStep& x = r.samples[j];
                m.real_tokens_processed += 1 + x.k;
                useful += 1 + x.k;
                if (config.mode == Mode::vanilla) pad += x.kv_padding;
                taus += (j ? "," : "") + std::to_string(x.tau);
            }
            led += std::string(i ? "," : "") + "{\"tau_list\":" + taus + "],\"tau_max\":" + std::to_string(r.tau_max) +
                   ",\"pad_writes\":" + std::to_string(pad) + ",\"useful_writes\":" + std::to_string(useful) + "}";
        }
        led += "]";
        if (config.mode == Mode::vanilla) m.pad_tokens_processed = m.total_input_padding + m.total_kv_padding;
        m.total_tokens_processed = m.real_tokens_processed + m.pad_tokens_processed;
    }
    if (m.decode_seconds > 0.0) m.tokens_per_second_decode = m.total_tokens_generated / m.decode_seconds;
    const double wall = m.prefill_seconds + m.decode_seconds;
    if (wall > 0.0) m.tokens_per_second_total = m.total_tokens_generated / wall;
    out.ledger_json = led;
    return out;
}

// JSON string: controls escaped, valid UTF-8 passed through, every byte that
// does not start a well-formed sequence replaced by U+FFFD (what the
// reference's dump does with error_handler_t::replace)
inline std::string json_string(const std::string& v) {
    std::string o = "\"";
    const size_t n = v.size();
    for (size_t i = 0; i < n;) {
        const unsigned char c = static_cast<unsigned char>(v[i]);
        if (c < 0x80) {
            switch (c) {
                case '"': o += "\\\""; break;
                case '\\': o += "\\\\"; break;
                case '\n': o += "\\n"; break;
                case '\t': o += "\\t"; break;
                case '\r': o += "\\r"; break;
                default:
                    if (c < 0x20) {
                        char buf[8];
                        std::snprintf(buf, sizeof buf, "\\u%04x", c);
                        o += buf;
                    } else {
                        o += static_cast<char>(c);
                    }
            }
            ++i;
            continue;
        }
        const size_t len = (c >= 0xC2 && c <= 0xDF) ? 2 : (c >= 0xE0 && c <= 0xEF) ? 3 : (c >= 0xF0 && c <= 0xF4) ? 4 : 0;
        bool ok = len > 0 && i + len <= n;
        for (size_t j = 1; ok && j < len; ++j) ok = (static_cast<unsigned char>(v[i + j]) & 0xC0) == 0x80;
        if (ok) {  // no overlong forms, surrogates or code points above U+10FFFF
            const unsigned char c1 = static_cast<unsigned char>(v[i + 1]);
            ok = !(c == 0xE0 && c1 < 0xA0) && !(c == 0xED && c1 > 0x9F) && !(c == 0xF0 && c1 < 0x90) &&
                 !(c == 0xF4 && c1 > 0x8F);
        }
        if (ok) {
            o.append(v, i, len);
            i += len;
        } else {
            o += "\xEF\xBF\xBD";
            ++i;
        }
    }
    return o + "\"";
}
inline std::string json_double(double v) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}
}  // namespace b200

// engine.cpp:206-289
inline DecodeResult decode_greedy(const std::vector<std::string>& prompts, const EngineConfig& config,
                                  const Model& target) {
    config.validate();
    if (static_cast<int>(prompts.size()) != config.batch_size)
        throw ContractError("prompt count does not match batch_size");
    EngineConfig g = config;
    g.mode = Mode::greedy;
    return b200::run_decode(prompts, g, target, nullptr);
}

// engine.cpp:291-528
inline DecodeResult decode_speculative(const std::vector<std::string>& prompts, const EngineConfig& config,
                                       const Model& target, const Model* draft) {
    config.validate();
    if (config.mode != Mode::vanilla && config.mode != Mode::ems)
        throw ConfigError("speculative decoding needs the vanilla or ems mode");
    if (static_cast<int>(prompts.size()) != config.batch_size)
        throw ContractError("prompt count does not match batch_size");
    return b200::run_decode(prompts, config, target, draft);
}

// engine.cpp:531-587: config, outputs, metrics, steps and the write ledger.
inline std::string results_json(const EngineConfig& config, const DecodeResult& result) {
    using b200::json_double;
    using b200::json_string;
    const RunMetrics& m = result.metrics;
    std::string o = "{\n  \"config\": {";
    o += "\"mode\": " + json_string(to_string(config.mode)) + ", \"predictor\": " +
         json_string(to_string(config.predictor)) + ", \"k\": " + std::to_string(config.k) +
         ", \"match_len\": " + std::to_string(config.match_len) + ", \"copy_len\": " + std::to_string(config.copy_len) +
         ", \"batch_size\": " + std::to_string(config.batch_size) +
         ", \"max_new_tokens\": " + std::to_string(config.max_new_tokens) +
         ", \"stop_on_eos\": " + (config.stop_on_eos ? "true" : "false") + ", \"seed\": " + std::to_string(config.seed) +
         ", \"synthetic_accuracy\": " + json_double(config.synthetic_accuracy) + "},\n  \"outputs\": [";
    for (size_t s = 0; s < result.generated_tokens.size(); ++s) {
        o += std::string(s ? ", " : "") + "{\"tokens\": [";
        for (size_t j = 0; j < result.generated_tokens[s].size(); ++j)
            o += std::string(j ? ", " : "") + std::to_string(result.generated_tokens[s][j]);
        o += "], \"text\": " + json_string(s < result.texts.size() ? result.texts[s] : std::string()) + "}";
    }
    o += "],\n  \"metrics\": {\"decode_steps\": " + std::to_string(m.decode_steps) + ", \"tokens_generated\": [";
    for (size_t s = 0; s < m.tokens_generated.size(); ++s)
        o += std::string(s ? ", " : "") + std::to_string(m.tokens_generated[s]);
    o += "], \"total_tokens_generated\": " + std::to_string(m.total_tokens_generated) +
         ", \"avg_acceptance_length\": " + json_double(m.avg_acceptance_length) +
         ", \"avg_padding_ratio\": " + json_double(m.avg_padding_ratio) +
         ", \"total_input_padding\": " + std::to_string(m.total_input_padding) +
         ", \"total_kv_padding\": " + std::to_string(m.total_kv_padding) +
         ", \"useful_kv_writes\": " + std::to_string(m.useful_kv_writes) +
         ", \"padding_kv_writes\": " + std::to_string(m.padding_kv_writes) +
         ", \"real_tokens_processed\": " + std::to_string(m.real_tokens_processed) +
         ", \"pad_tokens_processed\": " + std::to_string(m.pad_tokens_processed) +
         ", \"total_tokens_processed\": " + std::to_string(m.total_tokens_processed) +
         ", \"prefill_seconds\": " + json_double(m.prefill_seconds) +
         ", \"decode_seconds\": " + json_double(m.decode_seconds) +
         ", \"tokens_per_second_decode\": " + json_double(m.tokens_per_second_decode) +
         ", \"tokens_per_second_total\": " + json_double(m.tokens_per_second_total) + "},\n  \"steps\": [";
    for (size_t i = 0; i < result.steps.size(); ++i) {
        const StepRecord& r = result.steps[i];
        o += std::string(i ? ", " : "") + "{\"samples\": [";
        for (size_t j = 0; j < r.samples.size(); ++j) {
            const SampleStep& x = r.samples[j];
            o += std::string(j ? ", " : "") + "{\"sample\": " + std::to_string(x.sample) + ", \"k\": " +
                 std::to_string(x.k) + ", \"input_padding\": " + std::to_string(x.input_padding) +
                 ", \"tau\": " + std::to_string(x.tau) + ", \"kv_padding\": " + std::to_string(x.kv_padding) +
                 ", \"clipped\": " + (x.clipped ? "true" : "false") + "}";
        }
        o += "], \"tau_max\": " + std::to_string(r.tau_max) + ", \"delta_bar\": " + json_double(r.delta_bar) +
             ", \"r_bar\": " + json_double(r.r_bar) + "}";
    }
    o += "],\n  \"ledger\": " + (result.ledger_json.empty() ? std::string("[]") : result.ledger_json) + "\n}";
    return o;
}

}  // namespace specdec
