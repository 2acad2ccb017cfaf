// C ABI (include/specdec_b200.h) and the host-side validation that mirrors the
// reference's contracts before any device work is launched.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <string>
#include <vector>

#include "handles.h"

namespace sdb {

static std::atomic<int64_t> g_launches{0};
void note_launches(int64_t n) { g_launches += n; }

void set_device(int device) { CUDA_OK(cudaSetDevice(device)); }

int device_sm_count() {
    static std::mutex mu;
    static std::vector<int> sms;
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if ((int)sms.size() <= dev) sms.resize(dev + 1, 0);
    if (!sms[dev]) CUDA_OK(cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev));
    return sms[dev];
}

bool first_use_on_device(int key) {
    static std::mutex mu;
    static std::vector<std::pair<int, int>> seen;
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    for (auto& p : seen)
        if (p.first == dev && p.second == key) return false;
    seen.emplace_back(dev, key);
    return true;
}

bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("SD_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on != 0;
}

static int getenv_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

// ---------------------------------------------------------------- workspace
void Workspace::ensure(const Model& m, const Cache& c, int T) {
    if (T <= cap_tokens) return;
    int T2 = std::max(T, std::max(64, cap_tokens * 2));
    this->~Workspace();
    new (this) Workspace();
    const Config& cfg = m.cfg;
    size_t h = cfg.hidden(), mm = cfg.mlp(), V = cfg.vocab_size;
    d_tokens = (int32_t*)dmalloc(sizeof(int32_t) * T2);
    d_plans = (Plan*)dmalloc(sizeof(Plan) * T2);
    d_resid = (float*)dmalloc(sizeof(float) * T2 * h);
    d_tmp = (float*)dmalloc(sizeof(float) * T2 * 3 * h);
    d_tmp2 = (float*)dmalloc(sizeof(float) * T2 * (3 * h + mm));
    d_logits = (float*)dmalloc(sizeof(float) * T2 * V);
    d_argmax = (int32_t*)dmalloc(sizeof(int32_t) * T2);
    d_flag = (int32_t*)dmalloc(sizeof(int32_t) * 4);
    CUDA_OK(cudaMemset(d_flag, 0, sizeof(int32_t) * 4));
    if (m.precision == FP32_CHECK)
        d_scores = (float*)dmalloc(sizeof(float) * 2 * (size_t)T2 * cfg.num_heads * c.cap);
    d_segs = (SampleSeg*)dmalloc(sizeof(SampleSeg) * (size_t)c.B);
    d_qidx = (int32_t*)dmalloc(sizeof(int32_t) * T2);
    d_T = (int32_t*)dmalloc(sizeof(int32_t) * 4);
    segs_cap = c.B;
    cap_tokens = T2;
}

Workspace::~Workspace() {
    dfree(d_tokens);
    dfree(d_plans);
    dfree(d_resid);
    dfree(d_tmp);
    dfree(d_tmp2);
    dfree(d_logits);
    dfree(d_argmax);
    dfree(d_flag);
    dfree(d_scores);
    dfree(d_segs);
    dfree(d_qidx);
    dfree(d_T);
    free_fast_workspace(fast);
    fast = nullptr;
    cap_tokens = 0;
}

// -------------------------------------------------------------- construction
sd_model* create_model(const Config& cfg, int device, int precision, const float* host_weights) {
    SD_CHECK(cfg.num_layers >= 1, CONFIG, "num_layers must be >= 1");
    SD_CHECK(cfg.num_heads >= 1, CONFIG, "num_heads must be >= 1");
    SD_CHECK(cfg.head_dim >= 1, CONFIG, "head_dim must be >= 1");
    SD_CHECK(cfg.vocab_size >= 2, CONFIG, "vocab_size must be >= 2");
    SD_CHECK(cfg.max_positions >= 1, CONFIG, "max_positions must be >= 1");
    SD_CHECK(precision == FP32_CHECK || precision == BF16, CONFIG, "unknown precision");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(INTERNAL, "no CUDA device: the B200 kernels have no CPU fallback");
    SD_CHECK(device >= 0 && device < ndev, CONFIG, "device index out of range");
    cudaDeviceProp prop;
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        throw Error(INTERNAL, "device is sm_" + std::to_string(prop.major * 10 + prop.minor) +
                                  "; these kernels are built for sm_100a (B200) only");
    set_device(device);
    auto* h = new sd_model();
    try {
        Model& m = h->m;
        m.cfg = cfg;
        m.precision = precision;
        m.device = device;
        m.lay.build(cfg);
        CUDA_OK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
        int64_t hh = cfg.hidden(), mm = cfg.mlp();
        auto alloc = [&](size_t bytes) {
            void* p = dmalloc(bytes);
            m.allocations.push_back(p);
            m.weight_bytes += (int64_t)bytes;
            return p;
        };
        if (precision == FP32_CHECK) {
            m.w32 = (float*)alloc(sizeof(float) * (size_t)m.lay.total);
            if (host_weights) upload_weights_fp32(m, host_weights, h->st);
            else init_weights_fp32(m, h->st);
            note_launches(host_weights ? 0 : 2 + 17 * cfg.num_layers + 3);
        } else {
            m.vocab_pad = (cfg.vocab_size + 255) / 256 * 256;
            m.tok16 = (uint16_t*)alloc(2 * (size_t)cfg.vocab_size * hh);
            m.pos16 = (uint16_t*)alloc(2 * (size_t)cfg.max_positions * hh);
            m.lm16 = (uint16_t*)alloc(2 * (size_t)m.vocab_pad * hh);
            m.lnf_g = (float*)alloc(4 * hh);
            m.lnf_b = (float*)alloc(4 * hh);
            m.layers.resize(cfg.num_layers);
            for (FastLayer& f : m.layers) {
                f.wqkv = (uint16_t*)alloc(2 * (size_t)3 * hh * hh);
                f.wo = (uint16_t*)alloc(2 * (size_t)hh * hh);
                f.wfc = (uint16_t*)alloc(2 * (size_t)mm * hh);
                f.wproj = (uint16_t*)alloc(2 * (size_t)hh * mm);
                f.bqkv = (float*)alloc(4 * 3 * hh);
                f.bo = (float*)alloc(4 * hh);
                f.bfc = (float*)alloc(4 * mm);
                f.bproj = (float*)alloc(4 * hh);
                f.ln1_g = (float*)alloc(4 * hh);
                f.ln1_b = (float*)alloc(4 * hh);
                f.ln2_g = (float*)alloc(4 * hh);
                f.ln2_b = (float*)alloc(4 * hh);
            }
            if (host_weights) upload_weights_bf16(m, host_weights, h->st);
            else init_weights_bf16(m, h->st);
            build_fast_model(m);
            note_launches(host_weights ? 0 : 2 + 14 * cfg.num_layers + 3);
        }
        CUDA_OK(cudaStreamSynchronize(h->st));
    } catch (...) {
        delete h;
        throw;
    }
    return h;
}

// (re)allocate the device arena and descriptors for the current geometry
static void alloc_arena(sd_cache* h) {
    Cache& c = h->c;
    set_device(h->device);
    dfree(c.kv);
    dfree(c.d_committed);
    dfree(c.d_logical);
    dfree(c.d_pad);
    c.kv = nullptr;
    c.d_committed = c.d_logical = nullptr;
    c.d_pad = nullptr;
    size_t bytes = (size_t)c.L * 2 * c.B * c.heads * (size_t)c.cap * c.hd * c.elem_bytes;
    c.kv = dmalloc(bytes);
    CUDA_OK(cudaMemset(c.kv, 0, bytes));
    c.d_committed = (int32_t*)dmalloc(4 * (size_t)c.B);
    c.d_logical = (int32_t*)dmalloc(4 * (size_t)c.B);
    c.d_pad = (uint8_t*)dmalloc((size_t)c.B * c.cap);
    CUDA_OK(cudaMemset(c.d_committed, 0, 4 * (size_t)c.B));
    CUDA_OK(cudaMemset(c.d_logical, 0, 4 * (size_t)c.B));
    CUDA_OK(cudaMemset(c.d_pad, 0, (size_t)c.B * c.cap));
}

static sd_cache* new_cache(int layers, int batch, int capacity, int heads, int hd, int layout, int device,
                           int precision) {
    // CacheArena::CacheArena (kv_cache.cpp:78-88)
    SD_CHECK(layers >= 1 && batch >= 1 && capacity >= 1 && heads >= 1 && hd >= 1, CONFIG,
             "cache dimensions must be positive");
    SD_CHECK(layout == UNPAD || layout == PADDED, CONFIG, "unknown cache layout");
    SD_CHECK(precision == FP32_CHECK || precision == BF16, CONFIG, "unknown precision");
    auto* h = new sd_cache();
    try {
        Cache& c = h->c;
        c.layout = layout;
        c.L = layers;
        c.B = batch;
        c.cap = capacity;
        c.heads = heads;
        c.hd = hd;
        c.elem_bytes = precision == FP32_CHECK ? 4 : 2;
        h->device = device;
        h->precision = precision;
        h->lh.l = &c.ledger;
        alloc_arena(h);
        c.committed.assign(batch, 0);
        c.logical.assign(batch, 0);
        c.staged.assign(batch, 0);
        c.pad.assign((size_t)batch * capacity, 0);
        c.ledger.reset(batch);
    } catch (...) {
        delete h;
        throw;
    }
    return h;
}

sd_cache* create_cache(sd_model* mh, int batch, int capacity, int layout) {
    const Model& m = mh->m;
    set_device(m.device);
    sd_cache* h = new_cache(m.cfg.num_layers, batch, capacity, m.cfg.num_heads, m.cfg.head_dim, layout, m.device,
                            m.precision);
    h->c.model = &m;
    h->model = mh;
    return h;
}

sd_cache* create_cache_dims(int layers, int batch, int capacity, int kv_dim, int layout, int device, int precision) {
    set_device(device);
    return new_cache(layers, batch, capacity, 1, kv_dim, layout, device, precision);
}

// A dims-only arena meets its first model (Model::forward on a freshly built
// CacheArena, model.cpp:273-276): the depth and width must match; the arena
// takes the model's head split, element type and device.  Slots written
// through write_kv before that would have to move, so that is refused.
void bind_cache(sd_cache* h, sd_model* mh) {
    Cache& c = h->c;
    const Model& m = mh->m;
    if (h->model) return;
    SD_CHECK(c.heads * c.hd == m.cfg.hidden(), CONTRACT, "cache width does not match the model");
    SD_CHECK(c.L == m.cfg.num_layers, CONTRACT, "cache depth does not match the model");
    const int eb = m.precision == FP32_CHECK ? 4 : 2;
    if (c.heads != m.cfg.num_heads || c.elem_bytes != eb || h->device != m.device) {
        // masked holes are metadata only; stored rows would have to move
        SD_CHECK(!h->kv_stored, CONTRACT, "cache holds write_kv rows in a layout this model cannot read");
        c.heads = m.cfg.num_heads;
        c.hd = m.cfg.head_dim;
        c.elem_bytes = eb;
        h->device = m.device;
        h->precision = m.precision;
        alloc_arena(h);
    }
    c.model = &m;
    h->model = mh;
}

void reset_cache(sd_cache* h) {
    Cache& c = h->c;
    std::fill(c.committed.begin(), c.committed.end(), 0);
    std::fill(c.logical.begin(), c.logical.end(), 0);
    std::fill(c.staged.begin(), c.staged.end(), 0);
    std::fill(c.pad.begin(), c.pad.end(), 0);
    c.ledger.reset(c.B);
    cudaStream_t st = cache_stream(h);
    CUDA_OK(cudaMemsetAsync(c.d_committed, 0, 4 * (size_t)c.B, st));
    CUDA_OK(cudaMemsetAsync(c.d_logical, 0, 4 * (size_t)c.B, st));
    CUDA_OK(cudaMemsetAsync(c.d_pad, 0, (size_t)c.B * c.cap, st));
}

// ------------------------------------------------------------------ forward
static void sync_descriptors_to_device(sd_cache* h, cudaStream_t st) {
    Cache& c = h->c;
    CUDA_OK(cudaMemcpyAsync(c.d_committed, c.committed.data(), 4 * (size_t)c.B, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemcpyAsync(c.d_logical, c.logical.data(), 4 * (size_t)c.B, cudaMemcpyHostToDevice, st));
    if (c.layout == PADDED)
        CUDA_OK(cudaMemcpyAsync(c.d_pad, c.pad.data(), c.pad.size(), cudaMemcpyHostToDevice, st));
}

static void run_forward(sd_model* mh, sd_cache* h, int T, float* logits, int32_t* argmax) {
    Model& m = mh->m;
    cudaStream_t st = cache_stream(h);
    if (m.precision == FP32_CHECK) {
        forward_check(m, h->c, h->ws, T, true, st);
        note_launches(3 + 11 * (int64_t)m.cfg.num_layers + 3);
    } else {
        forward_fast(m, h->c, h->ws, T, logits != nullptr, st);
    }
    int32_t flag = 0;
    CUDA_OK(cudaMemcpyAsync(&flag, h->ws.d_flag, 4, cudaMemcpyDeviceToHost, st));
    if (argmax) CUDA_OK(cudaMemcpyAsync(argmax, h->ws.d_argmax, 4 * (size_t)T, cudaMemcpyDeviceToHost, st));
    if (logits)
        CUDA_OK(cudaMemcpyAsync(logits, h->ws.d_logits, 4 * (size_t)T * m.cfg.vocab_size,
                                cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (flag != 0) {
        CUDA_OK(cudaMemset(h->ws.d_flag, 0, 4));
        if (flag == 3) throw Error(CONTRACT, prefixed(CONTRACT, "token with an empty visible set"));
        throw Error(INTERNAL, "non-finite logit produced");
    }
}

void forward_planned_host(sd_model* mh, sd_cache* h, const int32_t* tokens, const Plan* plans, int n,
                          float* logits, int32_t* argmax) {
    Model& m = mh->m;
    Cache& c = h->c;
    const Config& cfg = m.cfg;
    set_device(m.device);
    // model.cpp:266-285
    SD_CHECK(n > 0, CONTRACT, "forward pass over zero tokens");
    check_idle(h);
    bind_cache(h, mh);
    SD_CHECK(c.model == &m && c.heads * c.hd == cfg.hidden(), CONTRACT, "cache width does not match the model");
    SD_CHECK(c.L == cfg.num_layers, CONTRACT, "cache depth does not match the model");
    for (int t = 0; t < n; ++t) {
        const Plan& p = plans[t];
        SD_CHECK(tokens[t] >= 0 && tokens[t] < cfg.vocab_size, CONTRACT, "token id out of vocabulary");
        SD_CHECK(p.sample >= 0 && p.sample < c.B, CONTRACT, "plan sample out of range");
        SD_CHECK(p.logical_pos >= 0, CONTRACT, "negative position");
        SD_CHECK(p.logical_pos < cfg.max_positions, CAPACITY,
                 "position " + std::to_string(p.logical_pos) + " exceeds max_positions " +
                     std::to_string(cfg.max_positions));
        if (!p.store) {  // CacheArena::mark_hole
            SD_CHECK(c.layout == PADDED, CONTRACT, "this cache layout has no masked holes");
            SD_CHECK(p.write_slot >= 0, CONTRACT, "cache position negative");
            SD_CHECK(p.write_slot < c.cap, CAPACITY,
                     "cache position " + std::to_string(p.write_slot) + " exceeds capacity " +
                         std::to_string(c.cap));
            c.pad[(size_t)p.sample * c.cap + p.write_slot] = 1;
            c.staged[p.sample] = std::max(c.staged[p.sample], p.write_slot + 1);
        }
    }
    // phase-1 write_kv checks and bookkeeping (kv_cache.cpp:93-103, 128-138, 203-213)
    for (int t = 0; t < n; ++t) {
        const Plan& p = plans[t];
        if (!p.store) continue;
        SD_CHECK(p.write_slot >= 0, CONTRACT, "cache position negative");
        SD_CHECK(p.write_slot < c.cap, CAPACITY,
                 "cache position " + std::to_string(p.write_slot) + " exceeds capacity " +
                     std::to_string(c.cap));
    }
    for (int t = 0; t < n; ++t) {
        const Plan& p = plans[t];
        if (!p.store) continue;
        if (c.layout == PADDED) c.pad[(size_t)p.sample * c.cap + p.write_slot] = 0;
        c.staged[p.sample] = std::max(c.staged[p.sample], p.write_slot + 1);
        c.ledger.note_useful(p.sample);  // once per slot, the layer-0 write (kv_cache.cpp:134-137)
    }
    // phase-2 gather checks (kv_cache.cpp:140-150): unpad reads stay below `written`
    if (c.layout == UNPAD)
        for (int t = 0; t < n; ++t)
            SD_CHECK(plans[t].write_slot < c.staged[plans[t].sample], CONTRACT, "read past the written extent");

    h->ws.ensure(m, c, n);
    cudaStream_t st = cache_stream(h);
    sync_descriptors_to_device(h, st);
    CUDA_OK(cudaMemcpyAsync(h->ws.d_tokens, tokens, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemcpyAsync(h->ws.d_plans, plans, sizeof(Plan) * (size_t)n, cudaMemcpyHostToDevice, st));
    run_forward(mh, h, n, logits, argmax);
}

void forward_ragged_host(sd_model* mh, sd_cache* h, const int32_t* tokens, const int32_t* counts, int batch,
                         const int32_t* slot_sample, const int32_t* slot_pos, float* logits,
                         int32_t* argmax) {
    Cache& c = h->c;
    SD_CHECK(batch >= 1, CONTRACT, "batch must have at least one sample");  // ragged.cpp:7
    SD_CHECK(batch <= c.B, CONTRACT, "batch has more samples than the cache");
    int n = 0;
    for (int s = 0; s < batch; ++s) {
        SD_CHECK(counts[s] >= 0, CONTRACT, "negative token count");
        n += counts[s];
    }
    std::vector<Plan> plans(n);
    int flat = 0;
    for (int s = 0; s < batch; ++s) {
        for (int o = 0; o < counts[s]; ++o, ++flat) {
            // restore_indices (ragged.cpp:19-36) collapses to this walk
            int expected = c.committed[s] + o;
            SD_CHECK(slot_sample[flat] == s && slot_pos[flat] == expected, CONTRACT,
                     "slot " + std::to_string(flat) + " does not continue its sample");
            plans[flat] = Plan{s, expected, expected, 1};
        }
    }
    forward_planned_host(mh, h, tokens, plans.data(), n, logits, argmax);
}

void commit_accepted_host(sd_cache* h, int s, int tau) {  // kv_cache.cpp:152-161
    check_idle(h);
    Cache& c = h->c;
    SD_CHECK(c.layout == UNPAD, CONTRACT, "not an unpad arena");
    SD_CHECK(s >= 0 && s < c.B, CONTRACT, "cache sample out of range");
    SD_CHECK(tau >= 1, CONTRACT, "commit needs tau >= 1");
    SD_CHECK(tau <= c.staged[s] - c.committed[s], CONTRACT, "commit exceeds the slots written this step");
    c.committed[s] += tau;
    c.logical[s] = c.committed[s];
    c.staged[s] = c.committed[s];
}

// --------------------------------------------------------------- verify step
// The step is split in two so that it can run asynchronously on a caller's
// stream: verify_step_enqueue validates on the host (before any state
// changes), stages the inputs in pinned memory and enqueues H2D -> pack ->
// forward -> accept [-> pad_fill] -> D2H on `st`; verify_step_finish waits
// for it, raises the device flags and applies the commit to the host mirrors
// and the ledger.  While a step is in flight the cache refuses other calls.
void verify_step_enqueue(sd_model* mh, sd_cache* h, const int32_t* last, const int32_t* counts,
                         const int32_t* drafts, const int32_t* budget, const int32_t* active, int stop_on_eos,
                         float* logits, cudaStream_t st) {
    SD_CHECK(!h->inflight.on, CONTRACT, "a verify step is already in flight on this cache");
    Model& m = mh->m;
    Cache& c = h->c;
    const Config& cfg = m.cfg;
    const int B = c.B;
    set_device(m.device);
    bind_cache(h, mh);
    // the cache must have been created for this model (model.cpp:273-276)
    SD_CHECK(c.model == &m && c.heads * c.hd == cfg.hidden(), CONTRACT, "cache width does not match the model");
    SD_CHECK(c.L == cfg.num_layers, CONTRACT, "cache depth does not match the model");
    // host validation (engine.cpp:427-444 / 408-426 and the forward contracts)
    int kmax = 0, nact = 0, ndraft = 0, base = -1;
    for (int s = 0; s < B; ++s) {
        SD_CHECK(counts[s] >= 0, CONTRACT, "negative draft count");
        ndraft += counts[s];
        if (!active[s]) {
            SD_CHECK(counts[s] == 0, CONTRACT, "inactive sample with drafts");
            continue;
        }
        nact++;
        kmax = std::max(kmax, counts[s]);
        SD_CHECK(budget[s] >= 1, CONTRACT, "active sample without generation budget");
        SD_CHECK(last[s] >= 0 && last[s] < cfg.vocab_size, CONTRACT, "token id out of vocabulary");
        if (c.layout == PADDED) {
            if (base < 0) base = c.committed[s];
            SD_CHECK(c.committed[s] == base, INTERNAL, "internal: aligned samples drifted apart");
        }
    }
    for (int i = 0; i < ndraft; ++i)
        SD_CHECK(drafts[i] >= 0 && drafts[i] < cfg.vocab_size, CONTRACT, "token id out of vocabulary");
    SD_CHECK(nact > 0, CONTRACT, "forward pass over zero tokens");
    int T = 0, max_kv = 0, max_q = 0;
    for (int s = 0; s < B; ++s) {
        if (!active[s]) continue;
        int n = c.layout == PADDED ? 1 + kmax : 1 + counts[s];
        int last_logical = (c.layout == PADDED ? c.logical[s] : c.committed[s]) + n - 1;
        int last_slot = (c.layout == PADDED ? base : c.committed[s]) + n - 1;
        SD_CHECK(last_logical < cfg.max_positions, CAPACITY,
                 "position " + std::to_string(last_logical) + " exceeds max_positions " +
                     std::to_string(cfg.max_positions));
        SD_CHECK(last_slot < c.cap, CAPACITY,
                 "cache position " + std::to_string(last_slot) + " exceeds capacity " + std::to_string(c.cap));
        T += n;
        max_kv = std::max(max_kv, last_slot + 1);
        max_q = std::max(max_q, n);
    }
    // device buffers: inputs [5B + kcap*B], scratch, outputs
    int kcap = std::max(kmax, 1);
    if (kcap > h->kcap || h->d_step == nullptr) {
        dfree(h->d_step);
        if (h->h_step) cudaFreeHost(h->h_step);
        h->kcap = std::max(kcap, 8);
        h->step_words = (size_t)B * (16 + 3 * (h->kcap + 1)) + 64;
        h->d_step = (int32_t*)dmalloc(4 * h->step_words);
        CUDA_OK(cudaMallocHost(&h->h_step, 4 * h->step_words));
    }
    int K1 = h->kcap + 1;
    int32_t* hs = h->h_step;
    int32_t* ds = h->d_step;
    // layout of the step block (words)
    size_t o_last = 0, o_counts = B, o_budget = 2 * B, o_active = 3 * B, o_drafts = 4 * B;
    size_t o_first = o_drafts + (size_t)B * h->kcap, o_doff = o_first + B, o_scal = o_doff + B;
    size_t o_tau = o_scal + 8, o_clip = o_tau + B, o_acc = o_clip + B;
    std::memcpy(hs + o_last, last, 4 * (size_t)B);
    std::memcpy(hs + o_counts, counts, 4 * (size_t)B);
    std::memcpy(hs + o_budget, budget, 4 * (size_t)B);
    std::memcpy(hs + o_active, active, 4 * (size_t)B);
    std::memcpy(hs + o_drafts, drafts, 4 * (size_t)ndraft);
    // the graph path below sizes its grids for B x (kcap + 1): allocate for that
    // bound up front (a reallocation would move buffers the StepArgs point at)
    h->ws.ensure(m, c, m.precision != FP32_CHECK && !logits && B * K1 <= 256 ? std::max(T, B * K1) : T);
    sync_descriptors_to_device(h, st);
    CUDA_OK(cudaMemcpyAsync(ds, hs, 4 * (o_drafts + ndraft), cudaMemcpyHostToDevice, st));
    StepArgs a{};
    a.B = B;
    a.cap = c.cap;
    a.layout = c.layout;
    a.stop_on_eos = stop_on_eos;
    a.acc_stride = K1;
    a.last = ds + o_last;
    a.counts = ds + o_counts;
    a.drafts = ds + o_drafts;
    a.budget = ds + o_budget;
    a.active = ds + o_active;
    a.committed = c.d_committed;
    a.logical = c.d_logical;
    a.pad = c.layout == PADDED ? c.d_pad : nullptr;
    a.tokens = h->ws.d_tokens;
    a.plans = h->ws.d_plans;
    a.segs = h->ws.d_segs;
    a.qidx = h->ws.d_qidx;
    a.first_row = ds + o_first;
    a.draft_off = ds + o_doff;
    a.scalars = ds + o_scal;
    a.argmax = h->ws.d_argmax;
    a.tau = ds + o_tau;
    a.accepted = ds + o_acc;
    a.clipped = ds + o_clip;
    // bf16, no logits: replay one CUDA graph of pack -> forward -> accept [->
    // pad_fill] whose grids are sized for the bound B x (kcap + 1) and read
    // the true token count on the device (like the session loop); the first
    // call runs eagerly so every lazily allocated buffer exists before capture
    const int T_up = B * K1;
    const bool graphable = m.precision != FP32_CHECK && !logits && T_up <= 256 && !profile_on() &&
                           getenv_int("SD_VERIFY_GRAPH", 1) != 0;
    const void* key[5] = {ds, h->ws.d_tokens, h->ws.fast, (const void*)(intptr_t)T_up, (const void*)&m};
    const int flags = (stop_on_eos ? 1 : 0) | (c.layout == PADDED ? 2 : 0);
    bool replay = false;
    if (graphable && h->vg_calls++ > 0) {
        if (!h->vgraph || h->vg_flags != flags || std::memcmp(h->vg_key, key, sizeof(key)) != 0) {
            if (h->vgraph) cudaGraphExecDestroy(h->vgraph);
            h->vgraph = nullptr;
            cudaGraph_t g;
            CUDA_OK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            launch_pack(a, st);
            DeviceBatch dbu{h->ws.d_segs, h->ws.d_qidx, ds + o_scal, T_up, c.cap, K1};
            forward_fast_dev(m, c, h->ws, dbu, 0, false, st);
            launch_accept(a, st);
            if (c.layout == PADDED) launch_pad_fill(a, c, st);
            CUDA_OK(cudaStreamEndCapture(st, &g));
            CUDA_OK(cudaGraphInstantiate(&h->vgraph, g, 0));
            CUDA_OK(cudaGraphDestroy(g));
            std::memcpy(h->vg_key, key, sizeof(key));
            h->vg_flags = flags;
        }
        CUDA_OK(cudaGraphLaunch(h->vgraph, st));
        replay = true;
    }
    if (!replay) {
        launch_pack(a, st);
        note_launches(1);
    }
    // run the forward (argmax always; logits on request)
    if (replay) {
    } else if (m.precision == FP32_CHECK) {
        forward_check(m, c, h->ws, T, true, st);
        note_launches(3 + 11 * (int64_t)cfg.num_layers + 3);
    } else if (T <= 256) {
        DeviceBatch db{h->ws.d_segs, h->ws.d_qidx, ds + o_scal, T, max_kv, max_q};
        forward_fast_dev(m, c, h->ws, db, 0, logits != nullptr, st);
    } else {
        forward_fast(m, c, h->ws, T, logits != nullptr, st);
    }
    if (!replay) {
        launch_accept(a, st);
        note_launches(1);
        if (c.layout == PADDED) {
            launch_pad_fill(a, c, st);
            note_launches(1);
        }
    }
    // device flag + outputs into the pinned step block (o_scal + 7 holds the flag)
    CUDA_OK(cudaMemcpyAsync(hs + o_scal + 7, h->ws.d_flag, 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(hs + o_tau, ds + o_tau, 4 * ((size_t)2 * B + (size_t)B * K1), cudaMemcpyDeviceToHost, st));
    if (logits)
        CUDA_OK(cudaMemcpyAsync(logits, h->ws.d_logits, 4 * (size_t)T * cfg.vocab_size, cudaMemcpyDeviceToHost, st));
    if (!h->done_ev) CUDA_OK(cudaEventCreateWithFlags(&h->done_ev, cudaEventDisableTiming));
    CUDA_OK(cudaEventRecord(h->done_ev, st));
    VerifyInflight& f = h->inflight;
    f.on = true;
    f.kmax = kmax;
    f.base = base;
    f.counts.assign(counts, counts + B);
    f.active.assign(active, active + B);
    f.o_tau = o_tau;
    f.o_clip = o_clip;
    f.o_acc = o_acc;
    f.o_flag = o_scal + 7;
    f.K1 = K1;
}

int verify_step_finish(sd_cache* h, int32_t* tau, int32_t* accepted, int32_t* clipped) {
    SD_CHECK(h->inflight.on, CONTRACT, "no verify step in flight on this cache");
    VerifyInflight& f = h->inflight;
    Cache& c = h->c;
    const int B = c.B, kmax = f.kmax, base = f.base, K1 = f.K1;
    const int32_t* counts = f.counts.data();
    const int32_t* active = f.active.data();
    const int32_t* hs = h->h_step;
    const size_t o_tau = f.o_tau, o_clip = f.o_clip, o_acc = f.o_acc;
    f.on = false;  // the step is consumed whatever happens below
    CUDA_OK(cudaEventSynchronize(h->done_ev));
    const int32_t flag = hs[f.o_flag];
    if (flag != 0) {
        CUDA_OK(cudaMemset(h->ws.d_flag, 0, 4));
        if (flag == 3) throw Error(CONTRACT, prefixed(CONTRACT, "token with an empty visible set"));
        throw Error(INTERNAL, "non-finite logit produced");
    }
    // outputs + host mirrors of the device-side commit
    int tmax = 0;
    for (int s = 0; s < B; ++s) {
        tau[s] = hs[o_tau + s];
        clipped[s] = hs[o_clip + s];
        int W = kmax + 1;
        for (int j = 0; j < W; ++j) accepted[s * W + j] = active[s] && j < tau[s] ? hs[o_acc + (size_t)s * K1 + j] : -1;
        tmax = std::max(tmax, tau[s]);
    }
    // the ledger step of one decode iteration (engine.cpp:398-487): opened here
    // unless the caller holds one open around this call
    const bool own_step = !c.ledger.open;
    if (own_step) c.ledger.begin_step();
    for (int s = 0; s < B; ++s) {
        if (!active[s]) continue;
        c.ledger.note_useful(s, 1 + counts[s]);  // the real input rows; PAD rows are holes
        if (c.layout == UNPAD) {
            c.committed[s] += tau[s];
            c.logical[s] = c.committed[s];
            c.staged[s] = c.committed[s];
        } else {
            for (int o = 0; o <= kmax; ++o) c.pad[(size_t)s * c.cap + base + o] = o <= counts[s] ? 0 : 1;
            for (int r = base + tau[s]; r < base + tmax; ++r) c.pad[(size_t)s * c.cap + r] = 1;
            c.ledger.note_padding(s, tmax - tau[s]);  // commit_padded's filler rows
            c.committed[s] = base + tmax;
            c.logical[s] += tau[s];
            c.staged[s] = c.committed[s];
        }
        c.ledger.note_tau(tau[s]);
    }
    if (own_step) c.ledger.end_step();
    return kmax;
}

int verify_step_host(sd_model* mh, sd_cache* h, const int32_t* last, const int32_t* counts,
                     const int32_t* drafts, const int32_t* budget, const int32_t* active, int stop_on_eos,
                     int32_t* tau, int32_t* accepted, int32_t* clipped, float* logits) {
    verify_step_enqueue(mh, h, last, counts, drafts, budget, active, stop_on_eos, logits, cache_stream(h));
    return verify_step_finish(h, tau, accepted, clipped);
}

void commit_prefill_host(sd_cache* h, const int32_t* samples, const int32_t* lens, int n) {  // kv_cache.cpp:237-267
        check_idle(h);
        Cache& c = h->c;
        SD_CHECK(c.layout == PADDED, CONTRACT, "not a padded grid");
        SD_CHECK(n >= 1, CONTRACT, "prefill commit needs matching sample and length lists");
        int rows = -1;
        for (int i = 0; i < n; ++i) {
            int s = samples[i], len = lens[i];
            SD_CHECK(s >= 0 && s < c.B, CONTRACT, "cache sample out of range");
            SD_CHECK(len >= 1, CONTRACT, "prompt length must be >= 1");
            SD_CHECK(c.committed[s] == 0, CONTRACT, "prefill commit on a non-empty sample");
            if (rows < 0) rows = c.staged[s];
            SD_CHECK(c.staged[s] == rows, CONTRACT, "prefill commit requires equally staged samples");
            SD_CHECK(len <= rows, CONTRACT, "prompt length exceeds staged rows");
            for (int r = 0; r < rows - len; ++r)
                SD_CHECK(c.pad[(size_t)s * c.cap + r], CONTRACT, "prefill left-pad row was not marked as a hole");
            for (int r = rows - len; r < rows; ++r)
                SD_CHECK(!c.pad[(size_t)s * c.cap + r], CONTRACT, "prefill prompt row was never written");
        }
        for (int i = 0; i < n; ++i) {
            c.committed[samples[i]] = rows;
            c.logical[samples[i]] = lens[i];
        }
}

void mark_hole_host(sd_cache* h, int s, int pos) {  // kv_cache.cpp:215-219
        check_idle(h);
        Cache& c = h->c;
        SD_CHECK(c.layout == PADDED, CONTRACT, "this cache layout has no masked holes");
        SD_CHECK(s >= 0 && s < c.B, CONTRACT, "cache sample out of range");
        SD_CHECK(pos >= 0, CONTRACT, "cache position negative");
        SD_CHECK(pos < c.cap, CAPACITY, "cache position " + std::to_string(pos) + " exceeds capacity " + std::to_string(c.cap));
        c.pad[(size_t)s * c.cap + pos] = 1;
        c.staged[s] = std::max(c.staged[s], pos + 1);
}

}  // namespace sdb

sd_model::~sd_model() {
    if (st) cudaStreamDestroy(st);
}
sd_cache::~sd_cache() {
    if (inflight.on && done_ev) cudaEventSynchronize(done_ev);  // never free buffers under a running step
    if (done_ev) cudaEventDestroy(done_ev);
    if (vgraph) cudaGraphExecDestroy(vgraph);
    sdb::dfree(d_step);
    if (h_step) cudaFreeHost(h_step);
}

// ===================================================================== C ABI
using namespace sdb;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return INTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return INTERNAL;
    }
}

Config to_cfg(const sd_model_config* c) {
    return Config{c->num_layers, c->num_heads, c->head_dim, c->vocab_size, c->max_positions, c->init_seed};
}

// SDCK v1 (model.cpp:143-221)
std::vector<float> read_sdck(const char* path, Config& cfg) {
    std::ifstream in(path, std::ios::binary);
    SD_CHECK(in.good(), IO, std::string("cannot open checkpoint: ") + path);
    auto rd = [&](void* p, size_t n, const char* what) {
        in.read((char*)p, (std::streamsize)n);
        SD_CHECK((size_t)in.gcount() == n, IO, std::string("checkpoint truncated while reading ") + what);
    };
    char magic[4];
    rd(magic, 4, "magic");
    SD_CHECK(std::memcmp(magic, "SDCK", 4) == 0, IO, std::string("not a model checkpoint: ") + path);
    uint32_t ver = 0;
    rd(&ver, 4, "version");
    SD_CHECK(ver == 1, IO, "unsupported checkpoint version " + std::to_string(ver));
    int32_t dims[5];
    rd(dims, sizeof dims, "dimensions");
    cfg = Config{dims[0], dims[1], dims[2], dims[3], dims[4], 0};
    rd(&cfg.init_seed, 8, "seed");
    SD_CHECK(cfg.num_layers >= 1, CONFIG, "num_layers must be >= 1");
    SD_CHECK(cfg.num_heads >= 1, CONFIG, "num_heads must be >= 1");
    SD_CHECK(cfg.head_dim >= 1, CONFIG, "head_dim must be >= 1");
    SD_CHECK(cfg.vocab_size >= 2, CONFIG, "vocab_size must be >= 2");
    SD_CHECK(cfg.max_positions >= 1, CONFIG, "max_positions must be >= 1");
    WeightLayout lay;
    lay.build(cfg);
    std::vector<float> w((size_t)lay.total);
    rd(w.data(), sizeof(float) * w.size(), "weights");
    char extra;
    in.read(&extra, 1);
    SD_CHECK(in.gcount() == 0, IO, std::string("checkpoint has trailing bytes: ") + path);
    return w;
}

std::vector<float> download_fp32(const sd_model* m) {
    SD_CHECK(m->m.precision == FP32_CHECK, CONTRACT, "fp32 weights exist only in the fp32 check mode");
    std::vector<float> w((size_t)m->m.lay.total);
    CUDA_OK(cudaSetDevice(m->m.device));
    CUDA_OK(cudaMemcpy(w.data(), m->m.w32, sizeof(float) * w.size(), cudaMemcpyDeviceToHost));
    return w;
}
}  // namespace

extern "C" {

const char* sd_last_error(void) { return g_err.c_str(); }
int64_t sd_kernel_launches(void) { return g_launches.load(); }

int sd_profile_enable(int on) {
    return guarded([&] { profile_enable(on != 0); });
}
int sd_profile_read(double* out, int kinds) {
    return guarded([&] { profile_read(out, kinds); });
}

int sd_config_validate(const sd_model_config* cfg) {
    return guarded([&] {
        SD_CHECK(cfg->num_layers >= 1, CONFIG, "num_layers must be >= 1");
        SD_CHECK(cfg->num_heads >= 1, CONFIG, "num_heads must be >= 1");
        SD_CHECK(cfg->head_dim >= 1, CONFIG, "head_dim must be >= 1");
        SD_CHECK(cfg->vocab_size >= 2, CONFIG, "vocab_size must be >= 2");
        SD_CHECK(cfg->max_positions >= 1, CONFIG, "max_positions must be >= 1");
    });
}

int sd_model_init(const sd_model_config* cfg, int device, int precision, sd_model** out) {
    return guarded([&] { *out = create_model(to_cfg(cfg), device, precision, nullptr); });
}

int sd_model_load(const char* path, int device, int precision, sd_model** out) {
    return guarded([&] {
        Config cfg;
        std::vector<float> w = read_sdck(path, cfg);
        *out = create_model(cfg, device, precision, w.data());
    });
}

int sd_model_save(const sd_model* m, const char* path) {
    return guarded([&] {
        std::vector<float> w = download_fp32(m);
        std::ofstream out(path, std::ios::binary);
        SD_CHECK(out.good(), IO, std::string("cannot open checkpoint for writing: ") + path);
        const Config& c = m->m.cfg;
        uint32_t ver = 1;
        int32_t dims[5] = {c.num_layers, c.num_heads, c.head_dim, c.vocab_size, c.max_positions};
        out.write("SDCK", 4);
        out.write((const char*)&ver, 4);
        out.write((const char*)dims, sizeof dims);
        out.write((const char*)&c.init_seed, 8);
        out.write((const char*)w.data(), (std::streamsize)(sizeof(float) * w.size()));
        SD_CHECK(out.good(), IO, std::string("checkpoint write failed: ") + path);
    });
}

int sd_model_checksum(const sd_model* m, uint64_t* out) {
    return guarded([&] {
        std::vector<float> w = download_fp32(m);
        uint64_t hash = 14695981039346656037ULL;  // FNV-1a, model.cpp:223-233
        const unsigned char* b = (const unsigned char*)w.data();
        for (size_t i = 0; i < w.size() * sizeof(float); ++i) {
            hash ^= b[i];
            hash *= 1099511628211ULL;
        }
        *out = hash;
    });
}

int sd_debug_model_compact(const sd_model* m) {
    if (!m) return -SD_CONTRACT;
    return m->m.fast && fast_model_compact(m->m) ? 1 : 0;
}

int sd_model_get_config(const sd_model* m, sd_model_config* out) {
    return guarded([&] {
        const Config& c = m->m.cfg;
        *out = sd_model_config{c.num_layers, c.num_heads, c.head_dim, c.vocab_size, c.max_positions, c.init_seed};
    });
}

int64_t sd_model_weight_bytes(const sd_model* m) { return m->m.weight_bytes; }

int sd_model_get_tensor(const sd_model* mh, int layer, int tensor, float* out, int64_t count) {
    return guarded([&] {  // model.hpp:81-87
        const Model& m = mh->m;
        const Config& c = m.cfg;
        const int64_t h = c.hidden(), mm = c.mlp();
        SD_CHECK(layer >= -1 && layer < c.num_layers, CONTRACT, "layer out of range");
        int64_t off32 = -1, n = 0;  // fp32 check mode: offset into the declaration-order blob
        const void* src = nullptr;  // bf16 mode: the stored tensor
        bool bf16 = true;
        if (layer < 0) {
            SD_CHECK(tensor >= 0 && tensor <= 4, CONTRACT, "unknown model tensor");
            const int64_t sizes[5] = {(int64_t)c.vocab_size * h, (int64_t)c.max_positions * h, h, h,
                                      (int64_t)c.vocab_size * h};
            const int64_t offs[5] = {m.lay.tok, m.lay.pos, m.lay.lnf_g, m.lay.lnf_b, m.lay.lm};
            n = sizes[tensor];
            off32 = offs[tensor];
            if (m.precision == BF16) {
                const void* p[5] = {m.tok16, m.pos16, m.lnf_g, m.lnf_b, m.lm16};
                src = p[tensor];
                bf16 = tensor == 0 || tensor == 1 || tensor == 4;
            }
        } else {
            SD_CHECK(tensor >= 0 && tensor <= 15, CONTRACT, "unknown layer tensor");
            const LayerOff& o = m.lay.layer[layer];
            const int64_t offs[16] = {o.ln1_g, o.ln1_b, o.wq, o.bq, o.wk, o.bk, o.wv, o.bv,
                                      o.wo, o.bo, o.ln2_g, o.ln2_b, o.w_fc, o.b_fc, o.w_proj, o.b_proj};
            const int64_t sizes[16] = {h, h, h * h, h, h * h, h, h * h, h, h * h, h, h, h, mm * h, mm, h * mm, h};
            n = sizes[tensor];
            off32 = offs[tensor];
            if (m.precision == BF16) {
                const FastLayer& f = m.layers[layer];
                const void* p[16] = {f.ln1_g, f.ln1_b, f.wqkv, f.bqkv, f.wqkv + h * h, f.bqkv + h,
                                     f.wqkv + 2 * h * h, f.bqkv + 2 * h, f.wo, f.bo, f.ln2_g, f.ln2_b,
                                     f.wfc, f.bfc, f.wproj, f.bproj};
                src = p[tensor];
                bf16 = tensor == 2 || tensor == 4 || tensor == 6 || tensor == 8 || tensor == 12 || tensor == 14;
            }
        }
        SD_CHECK(count == n, CONTRACT, "tensor size mismatch: expected " + std::to_string(n));
        CUDA_OK(cudaSetDevice(m.device));
        if (m.precision == FP32_CHECK) {
            CUDA_OK(cudaMemcpy(out, m.w32 + off32, sizeof(float) * (size_t)n, cudaMemcpyDeviceToHost));
        } else if (!bf16) {
            CUDA_OK(cudaMemcpy(out, src, sizeof(float) * (size_t)n, cudaMemcpyDeviceToHost));
        } else {
            std::vector<uint16_t> b((size_t)n);
            CUDA_OK(cudaMemcpy(b.data(), src, 2 * (size_t)n, cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < n; ++i) {
                uint32_t u = (uint32_t)b[i] << 16;
                std::memcpy(out + i, &u, 4);
            }
        }
    });
}

void sd_model_destroy(sd_model* m) {
    if (m) {
        cudaSetDevice(m->m.device);
        delete m;
    }
}

int sd_cache_create(const sd_model* m, int batch, int capacity, int layout, sd_cache** out) {
    return guarded([&] { *out = create_cache(const_cast<sd_model*>(m), batch, capacity, layout); });
}

int sd_cache_committed_len(const sd_cache* c, int s, int32_t* out) {
    return guarded([&] {
        SD_CHECK(s >= 0 && s < c->c.B, CONTRACT, "cache sample out of range");
        *out = c->c.committed[s];
    });
}
int sd_cache_logical_len(const sd_cache* c, int s, int32_t* out) {
    return guarded([&] {
        SD_CHECK(s >= 0 && s < c->c.B, CONTRACT, "cache sample out of range");
        *out = c->c.layout == UNPAD ? c->c.committed[s] : c->c.logical[s];
    });
}
int sd_cache_start_offset(const sd_cache* c, int s, int32_t* out) {  // kv_cache.cpp:116-120
    return guarded([&] {
        SD_CHECK(c->c.layout == UNPAD, CONTRACT, "not an unpad arena");
        SD_CHECK(s >= 0 && s < c->c.B, CONTRACT, "cache sample out of range");
        *out = s * c->c.cap;
    });
}
int sd_cache_commit_accepted(sd_cache* c, int s, int tau) {
    return guarded([&] { commit_accepted_host(c, s, tau); });
}

int sd_cache_get_lengths(const sd_cache* h, int32_t* committed, int32_t* start_offset) {
    return guarded([&] {  // kv_cache.hpp:109-110 for every sample at once
        const Cache& c = h->c;
        SD_CHECK(committed || start_offset, CONTRACT, "no output buffer");
        SD_CHECK(!start_offset || c.layout == UNPAD, CONTRACT, "start offsets exist for the unpad arena only");
        for (int s = 0; s < c.B; ++s) {
            if (committed) committed[s] = c.committed[s];
            if (start_offset) start_offset[s] = s * c.cap;
        }
    });
}

int sd_commit_accepted(sd_cache* h, const int32_t* taus) {
    return guarded([&] {  // UnpadArena::commit_accepted for every sample with tau > 0
        const Cache& c = h->c;
        SD_CHECK(c.layout == UNPAD, CONTRACT, "not an unpad arena");
        for (int s = 0; s < c.B; ++s)  // validate everything before any state changes (kv_cache.cpp:152-161)
            SD_CHECK(taus[s] >= 0 && taus[s] <= c.staged[s] - c.committed[s], CONTRACT,
                     "commit exceeds the slots written this step");
        for (int s = 0; s < c.B; ++s)
            if (taus[s] > 0) commit_accepted_host(h, s, taus[s]);
    });
}

int sd_cache_commit_prefill(sd_cache* h, const int32_t* samples, const int32_t* lens, int n) {
    return guarded([&] { commit_prefill_host(h, samples, lens, n); });
}

int sd_cache_commit_padded(sd_cache* h, const int32_t* samples, const int32_t* taus, int n) {
    return guarded([&] {  // kv_cache.cpp:269-314
        check_idle(h);
        Cache& c = h->c;
        SD_CHECK(c.layout == PADDED, CONTRACT, "not a padded grid");
        SD_CHECK(n >= 1, CONTRACT, "padded commit needs matching sample and tau lists");
        int tmax = 0;
        for (int i = 0; i < n; ++i) {
            SD_CHECK(taus[i] >= 1, CONTRACT, "commit needs tau >= 1");
            tmax = std::max(tmax, taus[i]);
        }
        c.ledger.check_tau(tmax);  // commit_padded notes every tau (kv_cache.cpp:312): a step must be open
        int base = -1;
        for (int i = 0; i < n; ++i) {
            int s = samples[i];
            SD_CHECK(s >= 0 && s < c.B, CONTRACT, "cache sample out of range");
            if (base < 0) base = c.committed[s];
            SD_CHECK(c.committed[s] == base, CONTRACT, "padded commit requires aligned samples");
            SD_CHECK(base + tmax <= c.cap, CAPACITY, "padded commit exceeds cache capacity");
            SD_CHECK(taus[i] <= c.staged[s] - base, CONTRACT, "commit exceeds the slots written this step");
            for (int r = base; r < base + taus[i]; ++r)
                SD_CHECK(!c.pad[(size_t)s * c.cap + r], CONTRACT, "accepted row was never written");
        }
        set_device(h->device);
        cudaStream_t st = cache_stream(h);
        // the filler rows of every sample and layer in ONE launch (kv_cache.cpp:295-307)
        std::vector<int32_t> rows(2 * (size_t)n);
        for (int i = 0; i < n; ++i) {
            rows[i] = samples[i];
            rows[n + i] = base + taus[i];
        }
        int32_t* d = (int32_t*)dmalloc(sizeof(int32_t) * rows.size());
        try {
            CUDA_OK(cudaMemcpyAsync(d, rows.data(), sizeof(int32_t) * rows.size(), cudaMemcpyHostToDevice, st));
            launch_zero_rows(c, d, d + n, n, base + tmax, st);
            note_launches(1);
            CUDA_OK(cudaStreamSynchronize(st));
        } catch (...) {
            dfree(d);
            throw;
        }
        dfree(d);
        for (int i = 0; i < n; ++i) {
            int s = samples[i];
            for (int r = base + taus[i]; r < base + tmax; ++r) {
                c.pad[(size_t)s * c.cap + r] = 1;
                c.ledger.note_padding(s);
            }
            c.committed[s] += tmax;
            c.logical[s] += taus[i];
            c.staged[s] = c.committed[s];
            c.ledger.note_tau(taus[i]);
        }
    });
}

int sd_cache_mark_hole(sd_cache* h, int s, int pos) {
    return guarded([&] { mark_hole_host(h, s, pos); });
}

int sd_cache_is_pad(const sd_cache* h, int s, int row, int32_t* out) {
    return guarded([&] {
        const Cache& c = h->c;
        SD_CHECK(c.layout == PADDED, CONTRACT, "not a padded grid");
        SD_CHECK(s >= 0 && s < c.B, CONTRACT, "cache sample out of range");
        SD_CHECK(row >= 0, CONTRACT, "cache position negative");
        SD_CHECK(row < c.cap, CAPACITY, "cache position " + std::to_string(row) + " exceeds capacity " + std::to_string(c.cap));
        *out = c.pad[(size_t)s * c.cap + row];
    });
}

int sd_cache_ledger(const sd_cache* c, int64_t* useful, int64_t* padding) {
    return guarded([&] {
        *useful = c->c.ledger.useful();
        *padding = c->c.ledger.padding();
    });
}

int sd_cache_gather_visible(const sd_cache* h, int s, int upto, int layer, float* k_out, float* v_out,
                            int32_t* count) {
    return guarded([&] {
        check_idle(h);
        const Cache& c = h->c;
        SD_CHECK(s >= 0 && s < c.B, CONTRACT, "cache sample out of range");
        SD_CHECK(layer >= 0 && layer < c.L, CONTRACT, "cache layer out of range");
        SD_CHECK(upto >= 0, CONTRACT, "cache position negative");
        SD_CHECK(upto < c.cap, CAPACITY, "cache position " + std::to_string(upto) + " exceeds capacity " + std::to_string(c.cap));
        if (c.layout == UNPAD) SD_CHECK(upto < c.staged[s], CONTRACT, "read past the written extent");
        set_device(h->device);
        int hidden = c.heads * c.hd, n = 0;
        std::vector<float> kh((size_t)(upto + 1) * c.hd), vh(kh.size());
        std::vector<uint16_t> kb(kh.size()), vb(kh.size());
        std::vector<int> rows;
        for (int r = 0; r <= upto; ++r)
            if (c.layout == UNPAD || !c.pad[(size_t)s * c.cap + r]) rows.push_back(r);
        for (int hd = 0; hd < c.heads; ++hd) {
            for (int w = 0; w < 2; ++w) {
                const char* src = (const char*)c.kv + c.kv_offset(layer, w, s, hd, 0) * c.elem_bytes;
                float* dst = w == 0 ? kh.data() : vh.data();
                if (c.elem_bytes == 4) {
                    CUDA_OK(cudaMemcpy(dst, src, sizeof(float) * kh.size(), cudaMemcpyDeviceToHost));
                } else {
                    uint16_t* tmp = w == 0 ? kb.data() : vb.data();
                    CUDA_OK(cudaMemcpy(tmp, src, 2 * kh.size(), cudaMemcpyDeviceToHost));
                    for (size_t i = 0; i < kh.size(); ++i) {
                        uint32_t u = (uint32_t)tmp[i] << 16;
                        std::memcpy(&dst[i], &u, 4);
                    }
                }
            }
            for (size_t j = 0; j < rows.size(); ++j) {
                std::memcpy(k_out + j * hidden + (size_t)hd * c.hd, kh.data() + (size_t)rows[j] * c.hd, 4 * (size_t)c.hd);
                std::memcpy(v_out + j * hidden + (size_t)hd * c.hd, vh.data() + (size_t)rows[j] * c.hd, 4 * (size_t)c.hd);
            }
        }
        n = (int)rows.size();
        *count = n;
    });
}

int sd_cache_create_dims(int num_layers, int batch, int capacity, int kv_dim, int layout, int device,
                         int precision, sd_cache** out) {
    return guarded([&] { *out = create_cache_dims(num_layers, batch, capacity, kv_dim, layout, device, precision); });
}

int sd_cache_write_kv(sd_cache* h, int s, int pos, int layer, const float* k_vec, const float* v_vec) {
    return guarded([&] {  // UnpadArena / PaddedGrid::write_kv (kv_cache.cpp:93-103, 128-138, 203-213)
        check_idle(h);
        Cache& c = h->c;
        SD_CHECK(s >= 0 && s < c.B, CONTRACT, "cache sample out of range");
        SD_CHECK(layer >= 0 && layer < c.L, CONTRACT, "cache layer out of range");
        SD_CHECK(pos >= 0, CONTRACT, "cache position negative");
        SD_CHECK(pos < c.cap, CAPACITY, "cache position " + std::to_string(pos) + " exceeds capacity " +
                                            std::to_string(c.cap));
        set_device(h->device);
        const size_t eb = c.elem_bytes, row = (size_t)c.hd * eb, pitch = (size_t)c.cap * c.hd * eb;
        const int kv_dim = c.heads * c.hd;
        std::vector<uint16_t> b16(eb == 2 ? (size_t)kv_dim : 0);
        for (int w = 0; w < 2; ++w) {
            const float* src = w == 0 ? k_vec : v_vec;
            const void* hsrc = src;
            if (eb == 2) {  // the bf16 arena stores round-to-nearest-even bf16
                for (int i = 0; i < kv_dim; ++i) {
                    uint32_t u;
                    std::memcpy(&u, &src[i], 4);
                    b16[i] = (u & 0x7fffffffu) > 0x7f800000u ? (uint16_t)((u >> 16) | 0x40)
                                                             : (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
                }
                hsrc = b16.data();
            }
            char* dst = (char*)c.kv + c.kv_offset(layer, w, s, 0, pos) * eb;
            CUDA_OK(cudaMemcpy2D(dst, pitch, hsrc, row, row, c.heads, cudaMemcpyHostToDevice));
        }
        h->kv_stored = true;
        if (layer == 0) {  // the slot is counted once, on its layer-0 write
            if (c.layout == PADDED) c.pad[(size_t)s * c.cap + pos] = 0;
            c.staged[s] = std::max(c.staged[s], pos + 1);
            c.ledger.note_useful(s);
        }
    });
}

// ---- WriteLedger (kv_cache.hpp:13-57) ----------------------------------------
int sd_ledger_create(int batch, sd_ledger** out) {
    return guarded([&] {
        SD_CHECK(batch >= 0, CONFIG, "ledger batch must be >= 0");
        auto* l = new sd_ledger();
        l->own.reset(batch);
        *out = l;
    });
}
void sd_ledger_destroy(sd_ledger* l) {
    if (l && l->l == &l->own) delete l;  // a cache's ledger view is owned by the cache
}
int sd_cache_ledger_handle(sd_cache* c, sd_ledger** out) {
    return guarded([&] { *out = &c->lh; });
}
int sd_ledger_note_useful(sd_ledger* l, int sample) {
    return guarded([&] { l->l->note_useful(sample); });
}
int sd_ledger_note_padding(sd_ledger* l, int sample) {
    return guarded([&] { l->l->note_padding(sample); });
}
int sd_ledger_begin_step(sd_ledger* l) {
    return guarded([&] { l->l->begin_step(); });
}
int sd_ledger_note_tau(sd_ledger* l, int tau) {
    return guarded([&] { l->l->note_tau(tau); });
}
int sd_ledger_end_step(sd_ledger* l) {
    return guarded([&] { l->l->end_step(); });
}
int sd_ledger_totals(const sd_ledger* l, int64_t* useful, int64_t* padding) {
    return guarded([&] {
        if (useful) *useful = l->l->useful();
        if (padding) *padding = l->l->padding();
    });
}
int sd_ledger_batch(const sd_ledger* l, int32_t* batch) {
    return guarded([&] { *batch = (int32_t)l->l->useful_by.size(); });
}
int sd_ledger_by_sample(const sd_ledger* l, int64_t* useful, int64_t* padding) {
    return guarded([&] {
        const Ledger& g = *l->l;
        if (useful) std::memcpy(useful, g.useful_by.data(), 8 * g.useful_by.size());
        if (padding) std::memcpy(padding, g.padding_by.data(), 8 * g.padding_by.size());
    });
}
int sd_ledger_num_steps(const sd_ledger* l, int64_t* n) {
    return guarded([&] { *n = (int64_t)l->l->steps.size(); });
}
int sd_ledger_step(const sd_ledger* l, int64_t i, int32_t* tau_list, int32_t cap, int32_t* n_tau, int32_t* tau_max,
                   int64_t* pad_writes, int64_t* useful_writes) {
    return guarded([&] {
        const Ledger& g = *l->l;
        SD_CHECK(i >= 0 && i < (int64_t)g.steps.size(), CONTRACT, "ledger step out of range");
        const LedgerStep& st = g.steps[(size_t)i];
        *n_tau = (int32_t)st.taus.size();
        for (int32_t j = 0; j < *n_tau && j < cap; ++j) tau_list[j] = st.taus[j];
        *tau_max = st.tau_max;
        *pad_writes = st.pad_writes;
        *useful_writes = st.useful_writes;
    });
}
// WriteLedger::dump_json (kv_cache.cpp:53-62): [{tau_list, tau_max, pad_writes,
// useful_writes}, ...] in nlohmann's compact key order (sorted keys).  len
// receives the full length; at most cap-1 bytes plus a NUL are written.
int sd_ledger_dump_json(const sd_ledger* l, char* buf, int64_t cap, int64_t* len) {
    return guarded([&] {
        std::string o = "[";
        bool first = true;
        for (const LedgerStep& st : l->l->steps) {
            o += first ? "{" : ",{";
            first = false;
            o += "\"pad_writes\":" + std::to_string(st.pad_writes) + ",\"tau_list\":[";
            for (size_t j = 0; j < st.taus.size(); ++j) o += (j ? "," : "") + std::to_string(st.taus[j]);
            o += "],\"tau_max\":" + std::to_string(st.tau_max) + ",\"useful_writes\":" +
                 std::to_string(st.useful_writes) + "}";
        }
        o += "]";
        *len = (int64_t)o.size();
        if (buf && cap > 0) {
            size_t n = std::min((size_t)cap - 1, o.size());
            std::memcpy(buf, o.data(), n);
            buf[n] = 0;
        }
    });
}
// padding_ratio (kv_cache.cpp:64-76): mean over steps of (tau_max - mean tau) / tau_max
int sd_ledger_padding_ratio(const sd_ledger* l, double* out) {
    return guarded([&] {
        const Ledger& g = *l->l;
        SD_CHECK(!g.steps.empty(), CONTRACT, "padding ratio undefined without steps");
        double sum = 0.0;
        for (const LedgerStep& st : g.steps) {
            double mean = 0.0;
            for (int32_t t : st.taus) mean += t;
            mean /= (double)st.taus.size();
            sum += ((double)st.tau_max - mean) / (double)st.tau_max;
        }
        *out = sum / (double)g.steps.size();
    });
}

int sd_cache_set_stream(sd_cache* c, void* stream) {
    return guarded([&] {
        check_idle(c);
        c->user_stream = (cudaStream_t)stream;
    });
}

void sd_cache_destroy(sd_cache* c) {
    if (c) {
        cudaSetDevice(c->device);
        delete c;
    }
}

int sd_restore_indices(const int32_t* counts, int batch, int flat, int32_t* sample, int32_t* pos) {
    return guarded([&] {  // ragged.cpp:19-36
        SD_CHECK(flat >= 0, CONTRACT, "flat index must be nonnegative");
        int s = 0, p = flat;
        for (int i = 0; i < batch; ++i) {
            if (p >= counts[i]) {
                s += 1;
                p -= counts[i];
            } else {
                break;
            }
        }
        SD_CHECK(s < batch, CONTRACT, "flat index " + std::to_string(flat) + " outside batch");
        *sample = s;
        *pos = p;
    });
}

int sd_forward(const sd_model* m, sd_cache* c, const int32_t* tokens, const int32_t* counts, int batch,
               const int32_t* slot_sample, const int32_t* slot_pos, float* logits, int32_t* argmax) {
    return guarded([&] {
        forward_ragged_host(const_cast<sd_model*>(m), c, tokens, counts, batch, slot_sample, slot_pos, logits, argmax);
    });
}

int sd_forward_planned(const sd_model* m, sd_cache* c, const int32_t* tokens, int n, const int32_t* sample,
                       const int32_t* logical, const int32_t* slot, const int32_t* store, float* logits,
                       int32_t* argmax) {
    return guarded([&] {
        std::vector<Plan> plans(n > 0 ? n : 0);
        for (int i = 0; i < n; ++i) plans[i] = Plan{sample[i], logical[i], slot[i], store[i] != 0};
        forward_planned_host(const_cast<sd_model*>(m), c, tokens, plans.data(), n, logits, argmax);
    });
}

int sd_decode(const sd_engine_config* cfg, sd_model* target, sd_model* draft, const int32_t* prompts,
              const int32_t* prompt_lens, int32_t* gen_tokens, int32_t* gen_counts, int32_t* rec, int64_t rec_cap,
              int64_t* n_rec, int64_t* ledger, double* timing) {
    return guarded([&] {
        decode_impl(*cfg, target, draft, prompts, prompt_lens, gen_tokens, gen_counts, rec, rec_cap, n_rec, ledger,
                    timing);
    });
}

int sd_draft_predict(sd_model* draft, const int32_t* context, int n, int k, int32_t* out) {
    return guarded([&] {
        SD_CHECK(n >= 0 && (n == 0 || context), CONTRACT, "draft prediction needs a context");
        const std::vector<int32_t> d = draft_predict_fresh(draft, std::vector<int32_t>(context, context + n), k);
        std::copy(d.begin(), d.end(), out);
    });
}

int sd_retrieval_predict(const int32_t* context, int n, int match_len, int copy_len, int32_t* out, int32_t* n_out) {
    return guarded([&] {
        const std::vector<int32_t> d = retrieval_predict(std::vector<int32_t>(context, context + n), match_len, copy_len);
        std::copy(d.begin(), d.end(), out);
        *n_out = (int32_t)d.size();
    });
}

int sd_synthetic_predict(sd_model* target, const int32_t* context, int n, int k, double accuracy, uint64_t step_seed,
                         int32_t* out) {
    return guarded([&] {
        const std::vector<int32_t> d =
            synthetic_predict_fresh(target, std::vector<int32_t>(context, context + n), k, accuracy, step_seed);
        std::copy(d.begin(), d.end(), out);
    });
}

int sd_verify_step(sd_model* m, sd_cache* c, const int32_t* last, const int32_t* counts, const int32_t* drafts,
                   const int32_t* budget, const int32_t* active, int stop_on_eos, int32_t* tau,
                   int32_t* accepted, int32_t* clipped, float* logits) {
    return guarded([&] {
        verify_step_host(m, c, last, counts, drafts, budget, active, stop_on_eos, tau, accepted, clipped, logits);
    });
}

int sd_verify_step_async(sd_model* m, sd_cache* c, const int32_t* last, const int32_t* counts, const int32_t* drafts,
                         const int32_t* budget, const int32_t* active, int stop_on_eos, void* stream) {
    return guarded([&] {
        set_device(m->m.device);
        verify_step_enqueue(m, c, last, counts, drafts, budget, active, stop_on_eos, nullptr,
                            stream ? (cudaStream_t)stream : cache_stream(c));
    });
}

int sd_verify_step_wait(sd_cache* c, int32_t* tau, int32_t* accepted, int32_t* clipped) {
    return guarded([&] {
        set_device(c->device);
        verify_step_finish(c, tau, accepted, clipped);
    });
}

}  // extern "C"
