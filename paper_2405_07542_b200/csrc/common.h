// Internal shared declarations for libspecdec_b200 (host C++ + CUDA).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

namespace sdb {

// Error taxonomy of the reference (common.hpp:13-34); the C-ABI maps each to
// its status code (include/specdec_b200.h).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
enum Status { OK = 0, CONFIG = 1, CAPACITY = 2, CONTRACT = 3, IO = 4, INTERNAL = 5 };

inline std::string prefixed(int code, const std::string& m) {
    static const char* p[] = {"", "config: ", "capacity: ", "contract: ", "io: ", ""};
    return std::string(p[code]) + m;
}
#define SD_CHECK(cond, code, msg)                                              \
    do {                                                                       \
        if (!(cond)) throw ::sdb::Error((code), ::sdb::prefixed((code), (msg))); \
    } while (0)
#define CUDA_OK(expr)                                                          \
    do {                                                                       \
        cudaError_t e__ = (expr);                                              \
        if (e__ != cudaSuccess)                                                \
            throw ::sdb::Error(::sdb::INTERNAL, std::string("cuda: ") + #expr +  \
                                                    ": " + cudaGetErrorString(e__)); \
    } while (0)

enum Precision { FP32_CHECK = 0, BF16 = 1 };
enum Layout { UNPAD = 0, PADDED = 1 };

struct Config {
    int32_t num_layers, num_heads, head_dim, vocab_size, max_positions;
    uint64_t init_seed;
    int hidden() const { return num_heads * head_dim; }
    int mlp() const { return 4 * hidden(); }
};

// Offsets (in elements) of every tensor in the reference declaration order
// (model.cpp:166-175).  The fp32 check mode stores exactly this flat layout.
struct LayerOff {
    int64_t ln1_g, ln1_b, wq, bq, wk, bk, wv, bv, wo, bo, ln2_g, ln2_b, w_fc, b_fc, w_proj, b_proj;
};
struct WeightLayout {
    int64_t tok, pos, lnf_g, lnf_b, lm, total;
    std::vector<LayerOff> layer;
    void build(const Config& c);
};

// Device-side bf16 weights for the performance mode: GEMM operands stay in
// the reference's row-major [out, in] (= K-major) layout; Q/K/V are fused into
// one [3h, h] operand; the LM head is zero-padded to a multiple of the GEMM
// M tile.  Biases / LayerNorm parameters stay fp32.
struct FastLayer {
    uint16_t *wqkv, *wo, *wfc, *wproj;  // bf16 bits
    float *bqkv, *bo, *bfc, *bproj, *ln1_g, *ln1_b, *ln2_g, *ln2_b;
};

struct Model {
    Config cfg;
    int precision = FP32_CHECK;
    int device = 0;
    WeightLayout lay;
    float* w32 = nullptr;        // check mode: all tensors fp32, declaration order
    // perf mode
    uint16_t* tok16 = nullptr;   // [V, h] bf16
    uint16_t* pos16 = nullptr;   // [P, h] bf16
    uint16_t* lm16 = nullptr;    // [V_pad, h] bf16
    float *lnf_g = nullptr, *lnf_b = nullptr;
    int vocab_pad = 0;
    std::vector<FastLayer> layers;
    std::vector<void*> allocations;
    int64_t weight_bytes = 0;
    struct FastModelState* fast = nullptr;  // TMA descriptors of the bf16 weights
    ~Model();
};
struct FastModelState;
struct FastWorkspace;
void free_fast_model(FastModelState* f);
void free_fast_workspace(FastWorkspace* f);
void build_fast_model(Model& m);
bool fast_model_compact(const Model& m);  // layer GEMMs as cluster split-K launches

// WriteLedger (kv_cache.hpp:13-57, kv_cache.cpp:11-76): KV slot writes per
// sample split into useful / padding, and the per-step grouping the engine
// opens around one verify step (begin_step / note_tau / end_step).  Checks and
// messages follow the reference; the per-step counters only move while a
// step is open.
struct LedgerStep {
    std::vector<int32_t> taus;
    int32_t tau_max = 0;
    int64_t pad_writes = 0, useful_writes = 0;
};
struct Ledger {
    std::vector<int64_t> useful_by, padding_by;
    std::vector<LedgerStep> steps;
    bool open = false;
    void reset(int batch) {
        useful_by.assign(batch, 0);
        padding_by.assign(batch, 0);
        steps.clear();
        open = false;
    }
    void note_useful(int s, int64_t n = 1) {
        SD_CHECK(s >= 0 && s < (int)useful_by.size(), CONTRACT, "ledger sample out of range");
        useful_by[s] += n;
        if (open) steps.back().useful_writes += n;
    }
    void note_padding(int s, int64_t n = 1) {
        SD_CHECK(s >= 0 && s < (int)padding_by.size(), CONTRACT, "ledger sample out of range");
        padding_by[s] += n;
        if (open) steps.back().pad_writes += n;
    }
    void begin_step() {
        SD_CHECK(!open, CONTRACT, "ledger step already open");
        steps.emplace_back();
        open = true;
    }
    void check_tau(int tau) const {
        SD_CHECK(open, CONTRACT, "note_tau outside a step");
        SD_CHECK(tau >= 1, CONTRACT, "acceptance length must be >= 1");
    }
    void note_tau(int tau) {
        check_tau(tau);
        steps.back().taus.push_back(tau);
        if (tau > steps.back().tau_max) steps.back().tau_max = tau;
    }
    void end_step() {
        SD_CHECK(open, CONTRACT, "no ledger step open");
        SD_CHECK(!steps.back().taus.empty(), CONTRACT, "ledger step closed without any acceptance length");
        open = false;
    }
    int64_t useful() const {
        int64_t t = 0;
        for (int64_t v : useful_by) t += v;
        return t;
    }
    int64_t padding() const {
        int64_t t = 0;
        for (int64_t v : padding_by) t += v;
        return t;
    }
};

// Per-sample KV arena.  K and V live in [L][2][B][heads][cap][head_dim]
// (head-major per sample so the attention kernel streams one contiguous
// extent per (sample, head)).  Slot coordinates follow the reference: sample s
// owns slots [s*cap, (s+1)*cap) (kv_cache.cpp:116-120).
struct Cache {
    int layout = UNPAD;
    int L = 0, B = 0, cap = 0, heads = 0, hd = 0;
    int elem_bytes = 4;            // 4 (check) / 2 (bf16)
    void* kv = nullptr;            // arena
    int32_t* d_committed = nullptr;  // committed_len per sample (slot/grid-row coords)
    int32_t* d_logical = nullptr;    // logical length (padded grid); == committed for unpad
    uint8_t* d_pad = nullptr;        // [B*cap] pad flags (padded grid)
    // host mirrors (the host validates every call exactly like the reference)
    std::vector<int32_t> committed, logical, staged;
    std::vector<uint8_t> pad;
    Ledger ledger;
    const Model* model = nullptr;
    ~Cache();
    size_t kv_offset(int layer, int which, int s, int head, int pos) const {
        return ((((size_t)layer * 2 + which) * B + s) * heads + head) * (size_t)cap * hd +
               (size_t)pos * hd;
    }
};

// A token's route through the forward pass (model.hpp:41-46 TokenPlan).
struct Plan {
    int32_t sample, logical_pos, write_slot, store;
};

// Per-sample ragged descriptor consumed by the attention kernel: the sample's
// query tokens are qidx[q_start .. q_start + n_q) of the packed stream and its
// visible KV extent is slots [0, kv_len) (each query still sees only slots
// <= its own write_slot).  `wide`: the sample's queries are one contiguous run
// of >= kWideMin tokens (a prompt chunk), attended by the 128-query prefill
// kernel instead of the 8-query verification kernel (host-planned forwards only).
struct SampleSeg {
    int q_start, n_q, kv_len, wide;
};

// Where a device-described batch lives (written by k_pack or uploaded by the
// host) and the host-side upper bounds the launch grids are sized for.
struct DeviceBatch {
    const SampleSeg* segs;
    const int32_t* qidx;
    const int32_t* dT;   // device token count
    int T_upper;         // grid bound for token-parallel kernels (<= 256)
    int max_kv_upper;    // bound on any sample's kv_len
    int max_q_upper;     // bound on any (non-wide) sample's query count
    int max_wide_q = 0;  // bound on a wide sample's query count (0: no wide samples)
};

// ---- device entry points (defined in the .cu files) -------------------------
void init_weights_fp32(Model& m, cudaStream_t st);
void init_weights_bf16(Model& m, cudaStream_t st);
void upload_weights_fp32(Model& m, const float* host, cudaStream_t st);  // load path
void upload_weights_bf16(Model& m, const float* host, cudaStream_t st);

// Scratch for one forward pass, grown on demand.
struct Workspace {
    int cap_tokens = 0;
    int device = 0;
    int32_t* d_tokens = nullptr;
    Plan* d_plans = nullptr;
    float* d_resid = nullptr;     // [T, h] fp32 residual stream
    float* d_tmp = nullptr;       // [T, max(3h, m)] fp32 (check mode activations)
    float* d_tmp2 = nullptr;      // [T, max(3h, m)]
    float* d_logits = nullptr;    // [T, V] fp32 (materialised when requested)
    int32_t* d_argmax = nullptr;  // [T]
    int32_t* d_flag = nullptr;    // non-finite logit flag
    float* d_scores = nullptr;    // check-mode attention scratch [T, heads, cap]
    FastWorkspace* fast = nullptr;  // bf16-mode buffers and TMA descriptors
    SampleSeg* d_segs = nullptr;    // [batch] ragged descriptors
    int32_t* d_qidx = nullptr;      // [T]
    int32_t* d_T = nullptr;         // device token count
    int segs_cap = 0;
    void ensure(const Model& m, const Cache& c, int T);
    ~Workspace();
};

// Run the whole-model forward over T planned tokens already on device.
// Writes argmax (always) and fp32 logits when want_logits.
void forward_check(const Model& m, Cache& c, Workspace& ws, int T, bool want_logits,
                   cudaStream_t st);

void* dmalloc(size_t bytes);
void dfree(void* p);

// Per-device facts and one-time setup.  Kernel attributes
// (cudaFuncSetAttribute) and the SM count belong to a device, so they are
// keyed on the CURRENT device, never cached process-wide.
int device_sm_count();
// true exactly once per (current device, key): the caller then runs the setup
bool first_use_on_device(int key);

}  // namespace sdb
