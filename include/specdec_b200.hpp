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
//
// Differences, all at the boundary: a Model lives on one GPU (precision
// SD_FP32_CHECK -- bit-exact with the reference -- unless SD_BF16 is asked
// for); a cache arena binds to the first Model that runs a forward over it
// (its device buffers are created then, the dimensions must match); K/V rows
// are written by the forward on the device (there is no host write_kv), and
// the ledger exposes the useful / padding totals.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "specdec_b200.h"

namespace specdec {

using TokenId = int32_t;
using TokenSequence = std::vector<TokenId>;
using LogitsRow = std::vector<float>;

namespace tok {
constexpr TokenId kBos = 0;
constexpr TokenId kEos = 1;
constexpr TokenId kPad = 2;
constexpr int kVocabSize = 259;
}  // namespace tok

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

// Argmax with ties toward the lowest id (model.cpp:34-41).
inline TokenId greedy_next(const LogitsRow& row) {
    if (row.empty()) throw ContractError("greedy_next on an empty row");
    TokenId best = 0;
    for (size_t i = 1; i < row.size(); ++i)
        if (row[i] > row[best]) best = static_cast<TokenId>(i);
    return best;
}

class Model;

// Read contract shared by both layouts (kv_cache.hpp:68-101).  The device
// arena is created when a Model first runs a forward over it.
class CacheArena {
public:
    CacheArena(int num_layers, int batch_size, int capacity, int kv_dim, int layout)
        : num_layers_(num_layers), batch_size_(batch_size), capacity_(capacity), kv_dim_(kv_dim), layout_(layout) {
        if (num_layers <= 0 || batch_size <= 0 || capacity <= 0 || kv_dim <= 0)
            throw ConfigError("cache dimensions must be positive");
    }
    virtual ~CacheArena() = default;
    CacheArena(const CacheArena&) = delete;
    CacheArena& operator=(const CacheArena&) = delete;

    int num_layers() const { return num_layers_; }
    int batch_size() const { return batch_size_; }
    int capacity() const { return capacity_; }
    int kv_dim() const { return kv_dim_; }

    int committed_len(int sample) const {
        check_sample(sample);
        if (!h_) return 0;
        int32_t v = 0;
        b200::check(sd_cache_committed_len(h_.get(), sample, &v));
        return v;
    }
    int logical_len(int sample) const {
        check_sample(sample);
        if (!h_) return 0;
        int32_t v = 0;
        b200::check(sd_cache_logical_len(h_.get(), sample, &v));
        return v;
    }
    virtual void mark_hole(int sample, int position) {
        b200::check(sd_cache_mark_hole(bound(), sample, position));
    }
    // Copies the visible real K/V rows [0, upto] of (sample, layer), ascending.
    int gather_visible(int sample, int upto, int layer, float* k_out, float* v_out) const {
        if (!h_) return 0;
        int32_t n = 0;
        b200::check(sd_cache_gather_visible(h_.get(), sample, upto, layer, k_out, v_out, &n));
        return n;
    }
    // Ledger totals (kv_cache.hpp:21-45): useful / padding slot writes.
    int64_t useful_writes() const { return totals().first; }
    int64_t padding_writes() const { return totals().second; }

    // The C handle (binds on first forward; see Model::forward).
    sd_cache* handle() const { return h_.get(); }
    void bind(const sd_model* m) {
        if (h_) return;
        sd_model_config cfg{};
        b200::check(sd_model_get_config(m, &cfg));
        if (cfg.num_layers != num_layers_ || cfg.num_heads * cfg.head_dim != kv_dim_)
            throw ContractError("cache dimensions do not match the model");
        sd_cache* c = nullptr;
        b200::check(sd_cache_create(m, batch_size_, capacity_, layout_, &c));
        h_.reset(c, sd_cache_destroy);
    }

protected:
    sd_cache* bound() const {
        if (!h_) throw ContractError("cache arena not bound to a model yet (run a forward first)");
        return h_.get();
    }
    void check_sample(int s) const {
        if (s < 0 || s >= batch_size_) throw ContractError("cache sample out of range");
    }
    std::pair<int64_t, int64_t> totals() const {
        int64_t u = 0, p = 0;
        if (h_) b200::check(sd_cache_ledger(h_.get(), &u, &p));
        return {u, p};
    }
    int num_layers_, batch_size_, capacity_, kv_dim_, layout_;
    std::shared_ptr<sd_cache> h_;
};

// EMS-SD layout (kv_cache.hpp:105-128).
class UnpadArena : public CacheArena {
public:
    UnpadArena(int num_layers, int batch_size, int capacity, int kv_dim)
        : CacheArena(num_layers, batch_size, capacity, kv_dim, SD_UNPAD) {}
    int start_offset(int sample) const {
        check_sample(sample);
        return sample * capacity_;  // kv_cache.cpp:116-120
    }
    void commit_accepted(int sample, int tau) { b200::check(sd_cache_commit_accepted(bound(), sample, tau)); }
};

// Vanilla (aligned) layout (kv_cache.hpp:133-168).
class PaddedGrid : public CacheArena {
public:
    PaddedGrid(int num_layers, int batch_size, int capacity, int kv_dim)
        : CacheArena(num_layers, batch_size, capacity, kv_dim, SD_PADDED) {}
    bool is_pad(int sample, int row) const {
        int32_t v = 0;
        b200::check(sd_cache_is_pad(bound(), sample, row, &v));
        return v != 0;
    }
    void commit_prefill(const std::vector<int>& samples, const std::vector<int>& prompt_lens) {
        if (samples.size() != prompt_lens.size()) throw ContractError("commit_prefill: mismatched lists");
        std::vector<int32_t> s(samples.begin(), samples.end()), l(prompt_lens.begin(), prompt_lens.end());
        b200::check(sd_cache_commit_prefill(bound(), s.data(), l.data(), static_cast<int>(s.size())));
    }
    void commit_padded(const std::vector<int>& samples, const std::vector<int>& taus) {
        if (samples.size() != taus.size()) throw ContractError("commit_padded: mismatched lists");
        std::vector<int32_t> s(samples.begin(), samples.end()), t(taus.begin(), taus.end());
        b200::check(sd_cache_commit_padded(bound(), s.data(), t.data(), static_cast<int>(s.size())));
    }
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
        cache.bind(h_.get());
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
        cache.bind(h_.get());
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

    sd_model* handle() const { return h_.get(); }

private:
    Model(sd_model* m, const ModelConfig& c) : h_(m, sd_model_destroy), config_(c) {}
    std::vector<LogitsRow> rows(const std::vector<float>& flat, int T) const {
        std::vector<LogitsRow> out(T);
        for (int i = 0; i < T; ++i)
            out[i].assign(flat.begin() + static_cast<size_t>(i) * config_.vocab_size,
                          flat.begin() + static_cast<size_t>(i + 1) * config_.vocab_size);
        return out;
    }
    std::shared_ptr<sd_model> h_;
    ModelConfig config_;
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

}  // namespace specdec
