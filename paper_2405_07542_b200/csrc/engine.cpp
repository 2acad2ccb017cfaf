// Host step driver: the decode loops of engine.cpp (decode_greedy 206-289,
// decode_speculative 291-489) re-created over the device verify step.  The
// per-step control flow, predictor calls, clipping rules and step records are
// the reference's; every forward, verification and commit runs on the GPU
// (verify_step_host -> k_pack / forward / k_accept / k_pad_fill).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <vector>

#include "handles.h"

namespace sdb {
namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

uint64_t splitmix_next(uint64_t& st) {  // rng.hpp:15-20
    uint64_t z = (st += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t mix_seed(uint64_t a, uint64_t b, uint64_t c) {  // rng.hpp:43-46
    uint64_t st = a ^ (b * 0xD1B54A32D192ED03ULL) ^ (c * 0x8CB92BA72F3D8DD7ULL);
    return splitmix_next(st);
}

}  // namespace

// predictors.cpp:39-59 (LLMA prompt lookup: rightmost earlier match)
std::vector<int32_t> retrieval_predict(const std::vector<int32_t>& ctx, int match_len, int copy_len) {
    SD_CHECK(match_len >= 1, CONTRACT, "match length must be >= 1");
    SD_CHECK(copy_len >= 1, CONTRACT, "copy length must be >= 1");
    int len = (int)ctx.size(), suffix = len - match_len;
    if (suffix <= 0) return {};
    for (int start = suffix - 1; start >= 0; --start) {
        bool match = true;
        for (int i = 0; i < match_len && match; ++i) match = ctx[start + i] == ctx[suffix + i];
        if (!match) continue;
        int from = start + match_len, take = std::min(copy_len, len - from);
        return std::vector<int32_t>(ctx.begin() + from, ctx.begin() + from + take);
    }
    return {};
}

namespace {

// predictors.cpp:9-37: greedy k-token rollout on a FRESH cache every call
// (the scratch cache is reset, which is observationally a fresh arena).
std::vector<int32_t> draft_predict(sd_model* draft, sd_cache* scratch, const std::vector<int32_t>& ctx, int k) {
    SD_CHECK(k >= 1, CONTRACT, "draft length must be >= 1");
    SD_CHECK(!ctx.empty(), CONTRACT, "draft prediction needs a context");
    int len = (int)ctx.size();
    SD_CHECK(len + k <= draft->m.cfg.max_positions, CAPACITY, "context plus draft length exceeds max_positions");
    reset_cache(scratch);
    std::vector<int32_t> zeros(len, 0), pos(len), am(len);
    for (int i = 0; i < len; ++i) pos[i] = i;
    int32_t cnt = len;
    forward_ragged_host(draft, scratch, ctx.data(), &cnt, 1, zeros.data(), pos.data(), nullptr, am.data());
    commit_accepted_host(scratch, 0, len);
    std::vector<int32_t> out;
    int32_t next = am[len - 1];
    out.push_back(next);
    for (int i = 1; i < k; ++i) {
        int32_t one = 1, p = scratch->c.committed[0], z = 0, a = 0;
        forward_ragged_host(draft, scratch, &next, &one, 1, &z, &p, nullptr, &a);
        commit_accepted_host(scratch, 0, 1);
        next = a;
        out.push_back(next);
    }
    return out;
}

struct State {
    std::vector<int32_t> tokens;
    int64_t generated = 0;
    bool finished = false;
};

// predictors.cpp:61-72: the target's own greedy rollout, each position kept
// with probability `accuracy` (SplitMix64 coins from the step seed) and
// otherwise replaced by the next id
void corrupt_rollout(std::vector<int32_t>& d, double accuracy, uint64_t step_seed, int vocab) {
    uint64_t rs = step_seed;
    for (int32_t& t : d) {
        const double u = (double)(splitmix_next(rs) >> 11) * 0x1.0p-53;
        if (u >= accuracy) t = (t + 1) % vocab;
    }
}

}  // namespace

// Stand-alone predictors (predictors.hpp:13-20) for the C ABI: a fresh
// one-sample arena per draft rollout, as the reference allocates one per call.
std::vector<int32_t> draft_predict_fresh(sd_model* draft, const std::vector<int32_t>& ctx, int k) {
    SD_CHECK(k >= 1, CONTRACT, "draft length must be >= 1");
    SD_CHECK(!ctx.empty(), CONTRACT, "draft prediction needs a context");
    SD_CHECK((int)ctx.size() + k <= draft->m.cfg.max_positions, CAPACITY,
             "context plus draft length exceeds max_positions");
    std::unique_ptr<sd_cache> scratch(create_cache(draft, 1, draft->m.cfg.max_positions, UNPAD));
    return draft_predict(draft, scratch.get(), ctx, k);
}
std::vector<int32_t> synthetic_predict_fresh(sd_model* target, const std::vector<int32_t>& ctx, int k,
                                             double accuracy, uint64_t step_seed) {
    SD_CHECK(accuracy >= 0.0 && accuracy < 1.0, CONFIG, "predictor accuracy must lie in [0, 1)");
    std::vector<int32_t> d = draft_predict_fresh(target, ctx, k);
    corrupt_rollout(d, accuracy, step_seed, target->m.cfg.vocab_size);
    return d;
}

struct Decoder {
    const sd_engine_config& e;
    sd_model* target;
    sd_model* draft;
    sd_cache* draft_scratch = nullptr;
    sd_cache* target_scratch = nullptr;

    std::vector<int32_t> predict(const State& st, int step, int s) {  // engine.cpp:173-188
        if (e.predictor == 1) return retrieval_predict(st.tokens, e.match_len, e.copy_len);
        if (e.predictor == 0) return draft_predict(draft, draft_scratch, st.tokens, e.k);
        SD_CHECK(e.synthetic_accuracy >= 0.0 && e.synthetic_accuracy < 1.0, CONFIG,
                 "predictor accuracy must lie in [0, 1)");
        std::vector<int32_t> d = draft_predict(target, target_scratch, st.tokens, e.k);  // predictors.cpp:61-72
        corrupt_rollout(d, e.synthetic_accuracy, mix_seed(e.seed, (uint64_t)step, (uint64_t)(e.sample_id_base + s)),
                        target->m.cfg.vocab_size);
        return d;
    }
    ~Decoder() {
        delete draft_scratch;
        delete target_scratch;
    }
};

}  // namespace sdb

namespace sdb {
int decode_impl(const sd_engine_config& e, sd_model* target, sd_model* draft, const int32_t* prompts,
                const int32_t* prompt_lens, int32_t* gen_tokens, int32_t* gen_counts, int32_t* rec,
                int64_t rec_cap, int64_t* n_rec, int64_t* ledger, double* timing) {
    // EngineConfig::validate (engine.cpp:48-58)
    if (e.predictor != 1) SD_CHECK(e.k >= 1, CONFIG, "k must be >= 1");
    SD_CHECK(e.match_len >= 1, CONFIG, "match_len must be >= 1");
    SD_CHECK(e.copy_len >= 1, CONFIG, "copy_len must be >= 1");
    SD_CHECK(e.batch_size >= 1, CONFIG, "batch_size must be >= 1");
    SD_CHECK(e.max_new_tokens >= 0, CONFIG, "max_new_tokens must be >= 0");
    SD_CHECK(e.synthetic_accuracy >= 0.0 && e.synthetic_accuracy < 1.0, CONFIG,
             "synthetic accuracy must lie in [0, 1)");
    const Config& tc = target->m.cfg;
    const int b = e.batch_size, V = tc.vocab_size;
    *n_rec = 0;
    ledger[0] = ledger[1] = 0;
    timing[0] = timing[1] = 0.0;
    std::vector<State> st(b);
    size_t at = 0;
    for (int s = 0; s < b; ++s) {
        SD_CHECK(prompt_lens[s] >= 1, CONTRACT, "empty prompt");
        st[s].tokens.assign(prompts + at, prompts + at + prompt_lens[s]);
        at += prompt_lens[s];
    }
    auto finish = [&] {
        for (int s = 0; s < b; ++s) {
            gen_counts[s] = (int32_t)st[s].generated;
            std::memcpy(gen_tokens + (size_t)s * e.max_new_tokens,
                        st[s].tokens.data() + st[s].tokens.size() - st[s].generated, 4 * st[s].generated);
        }
    };

    if (e.mode == 0) {  // decode_greedy (engine.cpp:206-289)
        for (int s = 0; s < b; ++s)
            SD_CHECK((int)st[s].tokens.size() + e.max_new_tokens <= tc.max_positions, CAPACITY,
                     "prompt plus generation budget exceeds max_positions");
        if (e.max_new_tokens == 0) return finish(), 0;
        std::unique_ptr<sd_cache> cache(create_cache(target, 1, tc.max_positions, UNPAD));
        for (int s = 0; s < b; ++s) {
            reset_cache(cache.get());
            State& S = st[s];
            int plen = (int)S.tokens.size();
            auto t0 = Clock::now();
            std::vector<int32_t> zeros(plen, 0), pos(plen), am(plen);
            for (int i = 0; i < plen; ++i) pos[i] = i;
            int32_t cnt = plen;
            forward_ragged_host(target, cache.get(), S.tokens.data(), &cnt, 1, zeros.data(), pos.data(), nullptr, am.data());
            commit_accepted_host(cache.get(), 0, plen);
            int32_t next = am[plen - 1];
            S.tokens.push_back(next);
            S.generated = 1;
            timing[0] += since(t0);
            t0 = Clock::now();
            while (S.generated < e.max_new_tokens && !(e.stop_on_eos && next == 1)) {
                int32_t one = 1, p = cache->c.committed[0], z = 0, a = 0;
                forward_ragged_host(target, cache.get(), &next, &one, 1, &z, &p, nullptr, &a);
                commit_accepted_host(cache.get(), 0, 1);
                next = a;
                S.tokens.push_back(next);
                S.generated += 1;
            }
            timing[1] += since(t0);
            ledger[0] += cache->c.ledger.useful();
        }
        return finish(), 0;
    }

    // decode_speculative (engine.cpp:291-489)
    SD_CHECK(e.mode == 1 || e.mode == 2, CONFIG, "speculative decoding needs the vanilla or ems mode");
    if (e.predictor == 0) {
        SD_CHECK(draft != nullptr, CONFIG, "draft predictor needs a draft model");
        SD_CHECK(draft->m.cfg.vocab_size == V, CONFIG, "draft and target vocabularies differ");
    }
    int reach = e.predictor == 1 ? e.copy_len : e.k;
    for (int s = 0; s < b; ++s) {
        int need = (int)st[s].tokens.size() + e.max_new_tokens + reach;
        SD_CHECK(need <= tc.max_positions, CAPACITY,
                 "prompt plus generation budget needs " + std::to_string(need) + " positions but the model has " +
                     std::to_string(tc.max_positions));
    }
    if (e.max_new_tokens == 0) return finish(), 0;
    bool aligned = e.mode == 1;
    std::unique_ptr<sd_cache> cache(create_cache(target, b, tc.max_positions, aligned ? PADDED : UNPAD));
    Decoder dec{e, target, draft};
    if (e.predictor == 0) dec.draft_scratch = create_cache(draft, 1, draft->m.cfg.max_positions, UNPAD);
    if (e.predictor == 2) dec.target_scratch = create_cache(target, 1, tc.max_positions, UNPAD);

    // prefill (engine.cpp:330-385)
    auto t0 = Clock::now();
    {
        std::vector<int32_t> flat, am;
        std::vector<Plan> plans;
        std::vector<int> last_row(b);
        int rows_needed = 0;
        for (auto& S : st) rows_needed = std::max(rows_needed, (int)S.tokens.size());
        for (int s = 0; s < b; ++s) {
            int len = (int)st[s].tokens.size(), holes = aligned ? rows_needed - len : 0;
            for (int r = 0; r < holes; ++r) mark_hole_host(cache.get(), s, r);
            for (int i = 0; i < len; ++i) {
                flat.push_back(st[s].tokens[i]);
                plans.push_back(Plan{s, i, holes + i, 1});
            }
            last_row[s] = (int)flat.size() - 1;
        }
        am.resize(flat.size());
        forward_planned_host(target, cache.get(), flat.data(), plans.data(), (int)flat.size(), nullptr, am.data());
        std::vector<int32_t> ids(b), lens(b);
        for (int s = 0; s < b; ++s) {
            ids[s] = s;
            lens[s] = (int)st[s].tokens.size();
        }
        if (aligned) {
            commit_prefill_host(cache.get(), ids.data(), lens.data(), b);
        } else {
            for (int s = 0; s < b; ++s) commit_accepted_host(cache.get(), s, lens[s]);
        }
        for (int s = 0; s < b; ++s) {
            int32_t first = am[last_row[s]];
            st[s].tokens.push_back(first);
            st[s].generated = 1;
            st[s].finished = st[s].generated >= e.max_new_tokens || (e.stop_on_eos && first == 1);
        }
    }
    timing[0] = since(t0);

    // decode loop (engine.cpp:391-489)
    t0 = Clock::now();
    std::vector<int32_t> last(b), counts(b), budget(b), active(b), tau(b), clipped(b), acc;
    std::vector<int32_t> drafts;
    for (int step = 0;; ++step) {
        int nact = 0;
        for (int s = 0; s < b; ++s) nact += !st[s].finished;
        if (nact == 0) break;
        drafts.clear();
        for (int s = 0; s < b; ++s) {
            active[s] = !st[s].finished;
            counts[s] = 0;
            if (!active[s]) continue;
            std::vector<int32_t> d = dec.predict(st[s], step, s);
            counts[s] = (int)d.size();
            drafts.insert(drafts.end(), d.begin(), d.end());
            last[s] = st[s].tokens.back();
            budget[s] = (int)(e.max_new_tokens - st[s].generated);
        }
        int kmax = 0;
        for (int s = 0; s < b; ++s) kmax = std::max(kmax, counts[s]);
        acc.assign((size_t)b * (kmax + 1), -1);
        verify_step_host(target, cache.get(), last.data(), counts.data(), drafts.data(), budget.data(),
                         active.data(), e.stop_on_eos, tau.data(), acc.data(), clipped.data(), nullptr);
        for (int s = 0; s < b; ++s) {
            if (!active[s]) continue;
            SD_CHECK(tau[s] >= 1, INTERNAL, "internal: empty acceptance");
            for (int j = 0; j < tau[s]; ++j) st[s].tokens.push_back(acc[(size_t)s * (kmax + 1) + j]);
            st[s].generated += tau[s];
            st[s].finished = st[s].generated >= e.max_new_tokens || (e.stop_on_eos && st[s].tokens.back() == 1);
            if (*n_rec < rec_cap) {
                int32_t* r = rec + *n_rec * 6;
                r[0] = step;
                r[1] = s;
                r[2] = counts[s];
                r[3] = tau[s];
                r[4] = clipped[s];
                r[5] = 0;
            }
            *n_rec += 1;
        }
    }
    timing[1] = since(t0);
    ledger[0] = cache->c.ledger.useful();
    ledger[1] = cache->c.ledger.padding();
    finish();
    return 0;
}
}  // namespace sdb
