// Exercises include/specdec_b200.hpp (the reference-shaped C++ layer) on the
// GPU: C1 config, fp32 check mode, a ragged prefill and two EMS verify steps
// driven exactly like engine.cpp:427-485 (concatenate_inputs ->
// restore_indices -> forward -> verify -> commit_accepted).  Prints one line
// per fact; tests/test_cpp_layer.py replays the same calls on the CPU
// oracle and compares (fp32 check mode is bit-exact).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "specdec_b200.hpp"

using namespace specdec;

static uint64_t fnv1a(const std::vector<float>& row) {
    uint64_t h = 0xcbf29ce484222325ULL;
    const unsigned char* p = reinterpret_cast<const unsigned char*>(row.data());
    for (size_t i = 0; i < row.size() * sizeof(float); ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

// One forward of per-sample inputs placed right after each sample's committed extent.
static std::vector<LogitsRow> step_forward(const Model& m, UnpadArena& arena, const std::vector<TokenSequence>& in,
                                           int tag) {
    RaggedBatch batch = ragged::concatenate_inputs(in);
    std::vector<TokenSlot> slots;
    for (int i = 0; i < batch.total_input_token_nums; ++i) {
        TokenSlot s = ragged::restore_indices(batch.token_nums_per_sample, i);
        s.original_sequence_position += arena.committed_len(s.original_batch_index);  // absolute position
        slots.push_back(s);
    }
    std::vector<LogitsRow> rows = m.forward(batch, arena, slots);
    for (size_t i = 0; i < rows.size(); ++i)
        std::printf("fwd %d %zu %llu %d\n", tag, i, (unsigned long long)fnv1a(rows[i]), greedy_next(rows[i]));
    return rows;
}

int main() {
    const ModelConfig cfg{};  // C1: the reference's default ModelConfig
    Model m = Model::init(cfg);
    std::printf("checksum %llu\n", (unsigned long long)m.weight_checksum());
    const int B = 3, cap = 64;
    UnpadArena arena(cfg.num_layers, B, cap, cfg.hidden());
    std::vector<TokenSequence> prompts = {{0, 72, 101, 108, 108, 111}, {0, 87, 111}, {0, 33, 34, 35, 36}};

    // prefill: the whole prompts, then commit them; the last row gives the first token
    std::vector<LogitsRow> rows = step_forward(m, arena, prompts, 0);
    std::vector<TokenId> last(B);
    size_t off = 0;
    for (int s = 0; s < B; ++s) {
        off += prompts[s].size();
        last[s] = greedy_next(rows[off - 1]);
        arena.commit_accepted(s, (int)prompts[s].size());
    }
    // two verify steps with fixed ragged drafts (sample 1 drafts nothing in step 1)
    const std::vector<std::vector<TokenSequence>> drafts = {{{5, 6}, {}, {7}}, {{9}, {10, 11, 12}, {13, 14}}};
    for (int step = 0; step < 2; ++step) {
        std::vector<TokenSequence> in(B);
        for (int s = 0; s < B; ++s) {
            in[s] = {last[s]};
            in[s].insert(in[s].end(), drafts[step][s].begin(), drafts[step][s].end());
        }
        rows = step_forward(m, arena, in, step + 1);
        off = 0;
        for (int s = 0; s < B; ++s) {
            std::vector<LogitsRow> mine(rows.begin() + off, rows.begin() + off + in[s].size());
            off += in[s].size();
            VerifyResult v = verify(mine, drafts[step][s]);
            arena.commit_accepted(s, v.tau);
            last[s] = v.accepted.back();
            std::printf("tau %d %d %d %d\n", step + 1, s, v.tau, arena.committed_len(s));
        }
    }
    std::printf("ledger %lld %lld\n", (long long)arena.ledger().useful_total(), (long long)arena.ledger().padding_total());
    // the array forms of the C ABI: all lengths at once, batched commit
    int32_t com[3], so[3];
    b200::check(sd_cache_get_lengths(arena.handle(), com, so));
    std::printf("lengths %d %d %d %d %d %d\n", com[0], com[1], com[2], so[0], so[1], so[2]);
    const int32_t too_many[3] = {0, 5, 0};  // nothing was staged since the last commit
    const int rc = sd_commit_accepted(arena.handle(), too_many);
    b200::check(sd_cache_get_lengths(arena.handle(), com, nullptr));
    std::printf("batched_commit_rejected %d %d %d %d\n", rc, com[0], com[1], com[2]);
    std::printf("start_offset %d\n", arena.start_offset(2));

    // the aligned layout through the same header: acceptance.cpp:125-147's
    // scripted trace (PAD filler rows 3 + 4)
    {
        PaddedGrid grid(cfg.num_layers, 2, 32, cfg.hidden());
        auto stage = [&](int sample, int row, int count, int logical) {
            std::vector<TokenId> toks(count, 5);
            std::vector<TokenPlan> plans;
            for (int i = 0; i < count; ++i) plans.push_back(TokenPlan{sample, logical + i, row + i, true});
            m.forward_planned(toks, plans, grid);
        };
        stage(0, 0, 1, 0);
        stage(1, 0, 1, 0);
        grid.commit_prefill({0, 1}, {1, 1});
        grid.ledger().begin_step();
        stage(0, 1, 6, 1);
        stage(1, 1, 3, 1);
        grid.commit_padded({0, 1}, {4, 1});
        grid.ledger().end_step();
        const long long after1 = grid.ledger().padding_total();
        grid.ledger().begin_step();
        stage(0, 5, 3, 5);
        stage(1, 5, 6, 2);
        grid.commit_padded({0, 1}, {2, 6});
        grid.ledger().end_step();
        std::printf("grid_padding %lld %lld %d %d %d\n", after1, (long long)grid.ledger().padding_total(),
                    grid.committed_len(0), grid.logical_len(1), grid.is_pad(1, 2) ? 1 : 0);
    }

    // error taxonomy: the reference's exception types come back
    try {
        ragged::restore_indices({1, 2}, 3);
        std::printf("restore_indices did not throw\n");
    } catch (const ContractError& e) {
        std::printf("contract_error_ok %s\n", std::strncmp(e.what(), "contract: ", 10) == 0 ? "prefixed" : e.what());
    }
    try {
        ModelConfig bad = cfg;
        bad.num_heads = 0;
        Model::init(bad);
        std::printf("bad config did not throw\n");
    } catch (const ConfigError&) {
        std::printf("config_error_ok\n");
    }
    try {
        arena.commit_accepted(0, cap);  // past the capacity
        std::printf("over-commit did not throw\n");
    } catch (const Error&) {
        std::printf("commit_error_ok\n");
    }
    return 0;
}
