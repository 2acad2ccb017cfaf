// Decode sessions: one prefilled batch that can run the speculative decode
// loop (engine.cpp:391-489) either
//   * device-resident: predictor, pack, forward, verify, clip and commit all
//     on the GPU, steps replayed from a captured CUDA graph, no host round
//     trip per step; or
//   * host-driven: the reference's loop shape, one sd_verify_step per step
//     with the predictor on the host (H2D drafts, D2H tau + accepted tokens).
// A session can be reset to its post-prefill state (rollback is metadata
// only: committed lengths, grid rows and pad flags), which is what lets a
// benchmark replay the same generation many times.
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "handles.h"

struct sd_session {
    sd_model* model = nullptr;
    std::unique_ptr<sd_cache> cache;
    // draft predictor (engine predictor 0): the draft model and its own
    // persistent per-sample cache, device draft commit lengths
    sd_model* draft = nullptr;
    std::unique_ptr<sd_cache> dcache;
    int32_t *dcommit = nullptr, *lsnap = nullptr;
    std::vector<int32_t> snap_dcommit;
    sd_engine_config e{};
    int B = 0, ctx_cap = 0, kcap = 0, max_steps = 0;
    // device state
    int32_t *ctx = nullptr, *ctx_len = nullptr, *gen = nullptr, *active = nullptr, *counts = nullptr,
            *drafts = nullptr, *n_active = nullptr, *step = nullptr, *log_k = nullptr, *log_tau = nullptr, *log_drafts = nullptr,
            *traj = nullptr, *first_row = nullptr, *draft_off = nullptr, *scalars = nullptr, *tau = nullptr,
            *accepted = nullptr, *clipped = nullptr;
    int traj_stride = 0;
    int32_t* h_flag = nullptr;  // pinned
    // post-prefill snapshot
    std::vector<int32_t> prompt_lens, first_tok, snap_committed, snap_logical, snap_active;
    std::vector<uint8_t> snap_pad;
    std::vector<std::vector<int32_t>> prompts;
    bool prefilled = false;
    // graph
    cudaGraphExec_t graph = nullptr;
    int graph_steps = 0;
    cudaGraphExec_t loop_graph = nullptr;  // WHILE-node graph of the whole loop
    bool loop_unsupported = false;
    std::vector<void*> allocs;
    ~sd_session() {
        if (graph) cudaGraphExecDestroy(graph);
        if (loop_graph) cudaGraphExecDestroy(loop_graph);
        for (void* p : allocs) sdb::dfree(p);
        if (h_flag) cudaFreeHost(h_flag);
    }
};

namespace sdb {
namespace {

int32_t* ialloc(sd_session* s, size_t n) {
    int32_t* p = (int32_t*)dmalloc(sizeof(int32_t) * (n ? n : 1));
    s->allocs.push_back(p);
    CUDA_OK(cudaMemset(p, 0, sizeof(int32_t) * (n ? n : 1)));
    return p;
}

StepArgs step_args(sd_session* s) {
    Cache& c = s->cache->c;
    Workspace& ws = s->cache->ws;
    StepArgs a{};
    a.B = s->B;
    a.cap = c.cap;
    a.layout = c.layout;
    a.ablation = s->e.mode == 3 ? 1 : s->e.mode == 4 ? 2 : 0;
    a.stop_on_eos = s->e.stop_on_eos;
    a.acc_stride = s->kcap + 1;
    a.last = nullptr;
    a.counts = s->counts;
    a.drafts = s->drafts;
    a.draft_stride = s->kcap;
    a.budget = nullptr;
    a.active = s->active;
    a.ctx = s->ctx;
    a.ctx_len = s->ctx_len;
    a.ctx_cap = s->ctx_cap;
    a.gen = s->gen;
    a.max_new = s->e.max_new_tokens;
    a.n_active = s->n_active;
    a.log_k = s->log_k;
    a.log_tau = s->log_tau;
    a.log_drafts = s->log_drafts;
    a.log_kcap = s->kcap;
    a.step = s->step;
    a.max_steps = s->max_steps;
    a.committed = c.d_committed;
    a.logical = c.d_logical;
    a.pad = c.layout == PADDED ? c.d_pad : nullptr;
    a.tokens = ws.d_tokens;
    a.plans = ws.d_plans;
    a.segs = ws.d_segs;
    a.qidx = ws.d_qidx;
    a.first_row = s->first_row;
    a.draft_off = s->draft_off;
    a.scalars = s->scalars;
    a.argmax = ws.d_argmax;
    a.tau = s->tau;
    a.accepted = s->accepted;
    a.clipped = s->clipped;
    return a;
}

DraftArgs draft_args(sd_session* s) {
    Workspace& dws = s->dcache->ws;
    DraftArgs d{};
    d.B = s->B;
    d.k = s->e.k;
    d.kcap = s->kcap;
    d.cap = s->dcache->c.cap;
    d.active = s->active;
    d.ctx = s->ctx;
    d.ctx_len = s->ctx_len;
    d.ctx_cap = s->ctx_cap;
    d.dcommit = s->dcommit;
    d.lsnap = s->lsnap;
    d.drafts = s->drafts;
    d.counts = s->counts;
    d.tau = s->tau;
    d.tokens = dws.d_tokens;
    d.plans = dws.d_plans;
    d.segs = dws.d_segs;
    d.qidx = dws.d_qidx;
    d.dT = dws.d_T;
    d.argmax = dws.d_argmax;
    return d;
}

// one device-resident verify step (fixed launch sequence, graph-capturable)
void device_step(sd_session* s, cudaStream_t st, unsigned long long cond = 0, bool has_cond = false) {
    Cache& c = s->cache->c;
    StepArgs a = step_args(s);
    a.cond = cond;
    a.has_cond = has_cond ? 1 : 0;
    if (s->e.predictor == 0) {  // k draft-model steps over the persistent draft cache
        DraftArgs d = draft_args(s);
        Workspace& dws = s->dcache->ws;
        DeviceBatch dbd{dws.d_segs, dws.d_qidx, dws.d_T, 2 * s->B, s->dcache->c.cap, 2};
        for (int j = 0; j < s->e.k; ++j) {
            launch_draft_pack(d, j, st);
            forward_fast_dev(s->draft->m, s->dcache->c, dws, dbd, 0, false, st);
            launch_draft_take(d, j, st);
        }
        note_launches(2 * s->e.k);
        launch_pack(a, st);
        DeviceBatch db{a.segs, a.qidx, a.scalars, s->B * (s->kcap + 1), c.cap, s->kcap + 1};
        forward_fast_dev(s->model->m, c, s->cache->ws, db, 0, false, st);
        launch_accept(a, st);
        if (c.layout == PADDED) launch_pad_fill(a, c, st);
        launch_draft_commit(d, st);
        note_launches(c.layout == PADDED ? 4 : 3);
        return;
    }
    PredictArgs p{};
    p.kind = s->e.predictor;
    p.match_len = s->e.match_len;
    p.copy_len = s->e.copy_len;
    p.k = s->e.k;
    p.vocab = s->model->m.cfg.vocab_size;
    p.seed = s->e.seed;
    p.id_base = s->e.sample_id_base;
    p.accuracy = s->e.synthetic_accuracy;
    p.traj = s->traj;
    p.traj_stride = s->traj_stride;
    launch_predict(a, p, st);
    launch_pack(a, st);
    DeviceBatch db{a.segs, a.qidx, a.scalars, s->B * (s->kcap + 1), c.cap, s->kcap + 1};
    forward_fast_dev(s->model->m, c, s->cache->ws, db, 0, false, st);
    launch_accept(a, st);
    int64_t n = 3;
    if (c.layout == PADDED) {
        launch_pad_fill(a, c, st);
        n++;
    }
    note_launches(n);
}

}  // namespace

sd_session* session_create(sd_model* m, const sd_engine_config& e, int capacity, sd_model* draft = nullptr) {
    SD_CHECK(m->m.precision == BF16, CONFIG, "sessions run the bf16 performance path");
    SD_CHECK(e.mode >= 1 && e.mode <= 4, CONFIG,
             "speculative decoding needs the vanilla, ems or an ablation mode (unpad_input, unpad_kv)");
    SD_CHECK(e.predictor >= 0 && e.predictor <= 2, CONFIG, "unknown predictor");
    if (e.predictor == 0) {
        SD_CHECK(draft != nullptr, CONFIG, "draft predictor needs a draft model");
        SD_CHECK(draft->m.precision == BF16, CONFIG, "the device draft rollout runs the bf16 path");
        SD_CHECK(draft->m.cfg.vocab_size == m->m.cfg.vocab_size, CONFIG, "draft and target vocabularies differ");
        SD_CHECK(draft->m.device == m->m.device, CONFIG, "draft and target must live on the same device");
        SD_CHECK(e.k >= 1, CONFIG, "draft length must be >= 1");
    }
    SD_CHECK(e.batch_size >= 1, CONFIG, "batch_size must be >= 1");  // engine.cpp:51-56
    SD_CHECK(e.max_new_tokens >= 0, CONFIG, "max_new_tokens must be >= 0");
    auto* s = new sd_session();
    try {
        s->model = m;
        s->e = e;
        s->B = e.batch_size;
        s->kcap = e.predictor == 1 ? e.copy_len : e.k;
        s->draft = e.predictor == 0 ? draft : nullptr;
        SD_CHECK(s->B * (s->kcap + 1) <= 256, CONFIG, "batch x (drafts + 1) must be <= 256 tokens per step");
        s->ctx_cap = capacity + 16;
        s->max_steps = e.max_new_tokens + 2;
        s->cache.reset(create_cache(m, s->B, capacity, e.mode == 1 || e.mode == 3 ? PADDED : UNPAD));
        int B = s->B;
        s->ctx = ialloc(s, (size_t)B * s->ctx_cap);
        s->ctx_len = ialloc(s, B);
        s->gen = ialloc(s, B);
        s->active = ialloc(s, B);
        s->counts = ialloc(s, B);
        s->drafts = ialloc(s, (size_t)B * s->kcap);
        s->n_active = ialloc(s, 4);
        s->step = ialloc(s, 4);
        s->log_k = ialloc(s, (size_t)s->max_steps * B);
        s->log_tau = ialloc(s, (size_t)s->max_steps * B);
        s->log_drafts = ialloc(s, (size_t)s->max_steps * B * std::max(1, s->kcap));
        s->first_row = ialloc(s, B);
        s->draft_off = ialloc(s, B);
        s->scalars = ialloc(s, 8);
        s->tau = ialloc(s, B);
        s->clipped = ialloc(s, B);
        s->accepted = ialloc(s, (size_t)B * (s->kcap + 1));
        CUDA_OK(cudaMallocHost(&s->h_flag, 16));
        s->cache->ws.ensure(m->m, s->cache->c, 256);
        ensure_fast_workspace(m->m, s->cache->c, s->cache->ws);
        if (s->draft) {
            s->dcache.reset(create_cache(draft, B, capacity, UNPAD));
            s->dcache->ws.ensure(draft->m, s->dcache->c, 256);
            ensure_fast_workspace(draft->m, s->dcache->c, s->dcache->ws);
            s->dcommit = ialloc(s, B);
            s->lsnap = ialloc(s, B);
        }
    } catch (...) {
        delete s;
        throw;
    }
    return s;
}

void session_reset(sd_session* s) {
    SD_CHECK(s->prefilled, CONTRACT, "session has not been prefilled");
    Cache& c = s->cache->c;
    cudaStream_t st = s->model->st;
    int B = s->B;
    c.committed = s->snap_committed;
    c.logical = s->snap_logical;
    c.staged = s->snap_committed;
    c.pad = s->snap_pad;
    CUDA_OK(cudaMemcpyAsync(c.d_committed, c.committed.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemcpyAsync(c.d_logical, c.logical.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, st));
    if (c.layout == PADDED)
        CUDA_OK(cudaMemcpyAsync(c.d_pad, c.pad.data(), c.pad.size(), cudaMemcpyHostToDevice, st));
    // after prefill the context holds prompt + the first generated token; a zero
    // budget returns before prefill (engine.cpp:314-317): prompt only, no steps
    const int first = s->e.max_new_tokens > 0 ? 1 : 0;
    std::vector<int32_t> len(B), gen(B, first);
    for (int b = 0; b < B; ++b) {
        len[b] = s->prompt_lens[b] + first;
        if (first)
            CUDA_OK(cudaMemcpyAsync(s->ctx + (size_t)b * s->ctx_cap + s->prompt_lens[b], &s->first_tok[b], 4,
                                    cudaMemcpyHostToDevice, st));
    }
    CUDA_OK(cudaMemcpyAsync(s->ctx_len, len.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemcpyAsync(s->gen, gen.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemcpyAsync(s->active, s->snap_active.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemsetAsync(s->step, 0, 4, st));
    CUDA_OK(cudaMemsetAsync(s->scalars, 0, 32, st));
    CUDA_OK(cudaMemsetAsync(s->log_tau, 0, 4 * (size_t)s->max_steps * B, st));
    CUDA_OK(cudaMemsetAsync(s->log_k, 0xff, 4 * (size_t)s->max_steps * B, st));
    if (s->draft)  // the draft cache keeps the prompt KV; later positions are rewritten
        CUDA_OK(cudaMemcpyAsync(s->dcommit, s->snap_dcommit.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaStreamSynchronize(st));
}

// engine.cpp:330-385 prefill through the chunked bf16 forward
void session_prefill(sd_session* s, const int32_t* prompts, const int32_t* lens) {
    Cache& c = s->cache->c;
    const Config& cfg = s->model->m.cfg;
    int B = s->B;
    bool aligned = c.layout == PADDED;
    int rows_needed = 0;
    s->prompts.assign(B, {});
    s->prompt_lens.assign(B, 0);
    size_t at = 0;
    for (int b = 0; b < B; ++b) {
        SD_CHECK(lens[b] >= 1, CONTRACT, "empty prompt");
        s->prompts[b].assign(prompts + at, prompts + at + lens[b]);
        s->prompt_lens[b] = lens[b];
        at += lens[b];
        rows_needed = std::max(rows_needed, lens[b]);
        int reach = s->kcap;
        SD_CHECK(lens[b] + s->e.max_new_tokens + reach <= cfg.max_positions, CAPACITY,
                 "prompt plus generation budget exceeds max_positions");
        SD_CHECK(lens[b] + s->e.max_new_tokens + reach <= c.cap, CAPACITY,
                 "prompt plus generation budget exceeds the cache capacity");
        SD_CHECK(lens[b] + s->e.max_new_tokens + reach + 1 <= s->ctx_cap, CAPACITY, "context buffer too small");
    }
    // the prefill may grow the workspaces (Workspace::ensure reallocates the
    // token / plan / partial buffers), and the captured graphs bake in their
    // pointers: drop them so the next run recaptures against the live buffers
    if (s->graph) CUDA_OK(cudaGraphExecDestroy(s->graph));
    if (s->loop_graph) CUDA_OK(cudaGraphExecDestroy(s->loop_graph));
    s->graph = nullptr;
    s->loop_graph = nullptr;
    s->graph_steps = 0;
    s->loop_unsupported = false;
    reset_cache(s->cache.get());
    if (s->e.max_new_tokens == 0) {  // engine.cpp:314-317: nothing to prefill or decode
        for (int b = 0; b < B; ++b)
            CUDA_OK(cudaMemcpy(s->ctx + (size_t)b * s->ctx_cap, s->prompts[b].data(), 4 * (size_t)lens[b],
                               cudaMemcpyHostToDevice));
        s->first_tok.assign(B, 0);
        s->snap_active.assign(B, 0);
        if (s->draft) {
            reset_cache(s->dcache.get());
            s->snap_dcommit.assign(B, 0);
        }
        s->snap_committed = c.committed;
        s->snap_logical = c.logical;
        s->snap_pad = c.pad;
        s->prefilled = true;
        session_reset(s);
        return;
    }
    std::vector<int32_t> flat, am;
    std::vector<Plan> plans;
    std::vector<int> last_row(B);
    for (int b = 0; b < B; ++b) {
        int len = lens[b], holes = aligned ? rows_needed - len : 0;
        for (int r = 0; r < holes; ++r) mark_hole_host(s->cache.get(), b, r);
        for (int i = 0; i < len; ++i) {
            flat.push_back(s->prompts[b][i]);
            plans.push_back(Plan{b, i, holes + i, 1});
        }
        last_row[b] = (int)flat.size() - 1;
    }
    am.resize(flat.size());
    forward_planned_host(s->model, s->cache.get(), flat.data(), plans.data(), (int)flat.size(), nullptr, am.data());
    std::vector<int32_t> ids(B), pl(B);
    for (int b = 0; b < B; ++b) {
        ids[b] = b;
        pl[b] = lens[b];
    }
    if (aligned) commit_prefill_host(s->cache.get(), ids.data(), pl.data(), B);
    else
        for (int b = 0; b < B; ++b) commit_accepted_host(s->cache.get(), b, lens[b]);
    s->first_tok.assign(B, 0);
    s->snap_active.assign(B, 0);
    for (int b = 0; b < B; ++b) {
        s->first_tok[b] = am[last_row[b]];
        bool fin = 1 >= s->e.max_new_tokens || (s->e.stop_on_eos && s->first_tok[b] == 1);
        s->snap_active[b] = fin ? 0 : 1;
        CUDA_OK(cudaMemcpy(s->ctx + (size_t)b * s->ctx_cap, s->prompts[b].data(), 4 * (size_t)lens[b],
                           cudaMemcpyHostToDevice));
    }
    if (s->draft) {  // the draft model prefills the same prompts into its own cache
        const Config& dcfg = s->draft->m.cfg;
        std::vector<Plan> dplans;
        for (int b = 0; b < B; ++b) {
            SD_CHECK(lens[b] + s->e.max_new_tokens + s->e.k <= dcfg.max_positions, CAPACITY,
                     "prompt plus generation budget exceeds the draft model's max_positions");
            for (int i = 0; i < lens[b]; ++i) dplans.push_back(Plan{b, i, i, 1});
        }
        reset_cache(s->dcache.get());
        std::vector<int32_t> dam(flat.size());
        forward_planned_host(s->draft, s->dcache.get(), flat.data(), dplans.data(), (int)flat.size(), nullptr,
                             dam.data());
        for (int b = 0; b < B; ++b) commit_accepted_host(s->dcache.get(), b, lens[b]);
        s->snap_dcommit.assign(lens, lens + B);
    }
    s->snap_committed = c.committed;
    s->snap_logical = c.logical;
    s->snap_pad = c.pad;
    s->prefilled = true;
    session_reset(s);
}

void session_set_trajectory(sd_session* s, const int32_t* traj, int stride) {
    SD_CHECK(stride >= s->e.max_new_tokens + s->e.k, CONTRACT, "trajectory shorter than budget + k");
    if (!s->traj || s->traj_stride < stride) {
        s->traj = ialloc(s, (size_t)s->B * stride);
    }
    s->traj_stride = stride;
    CUDA_OK(cudaMemcpy(s->traj, traj, 4 * (size_t)s->B * stride, cudaMemcpyHostToDevice));
}

// device-resident loop; returns decode steps, GPU ms (events on the stream)
int session_run(sd_session* s, int use_graph, int graph_steps, float* gpu_ms) {
    SD_CHECK(s->prefilled, CONTRACT, "session has not been prefilled");
    SD_CHECK(s->e.predictor != 2 || s->traj, CONTRACT, "synthetic predictor needs a trajectory");
    cudaStream_t st = s->model->st;
    set_device(s->model->m.device);
    prepare_fast_kernels();
    if (graph_steps < 1) graph_steps = 8;
    if (use_graph && graph_steps == 8 && !s->loop_graph && !s->loop_unsupported) {
        // the whole loop as one graph: a WHILE conditional node whose body is
        // one verify step; k_accept sets the condition on the device
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ex = nullptr;
        bool ok = cudaGraphCreate(&g, 0) == cudaSuccess;
        cudaGraphConditionalHandle h{};
        ok = ok && cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        ok = ok && cudaGraphAddNode(&node, g, nullptr, 0, &cp) == cudaSuccess;
        if (ok) {
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            CUDA_OK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
            device_step(s, st, (unsigned long long)h, true);
            CUDA_OK(cudaStreamEndCapture(st, &body));
            ok = cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();  // clear a soft failure (old driver): fall back to replayed batches
        if (ok) s->loop_graph = ex;
        else s->loop_unsupported = true;
    }
    if (use_graph && s->loop_graph) {
        cudaEvent_t e0, e1;
        CUDA_OK(cudaEventCreate(&e0));
        CUDA_OK(cudaEventCreate(&e1));
        CUDA_OK(cudaEventRecord(e0, st));
        CUDA_OK(cudaGraphLaunch(s->loop_graph, st));
        CUDA_OK(cudaEventRecord(e1, st));
        CUDA_OK(cudaMemcpyAsync(s->h_flag + 1, s->step, 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaEventSynchronize(e1));
        CUDA_OK(cudaStreamSynchronize(st));
        float ms = 0.0f;
        CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (gpu_ms) *gpu_ms = ms;
        int32_t flag = 0, cap_err = 0;
        CUDA_OK(cudaMemcpy(&flag, s->cache->ws.d_flag, 4, cudaMemcpyDeviceToHost));
        CUDA_OK(cudaMemcpy(&cap_err, s->scalars + 4, 4, cudaMemcpyDeviceToHost));
        SD_CHECK(flag == 0, INTERNAL, "non-finite logit produced");
        SD_CHECK(cap_err == 0, CAPACITY, "padded grid outgrew the cache capacity during the device loop");
        return s->h_flag[1];
    }
    if (use_graph && (!s->graph || s->graph_steps != graph_steps)) {
        if (s->graph) cudaGraphExecDestroy(s->graph);
        s->graph = nullptr;
        cudaGraph_t g;
        CUDA_OK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < graph_steps; ++i) device_step(s, st);
        CUDA_OK(cudaStreamEndCapture(st, &g));
        CUDA_OK(cudaGraphInstantiate(&s->graph, g, 0));
        CUDA_OK(cudaGraphDestroy(g));
        s->graph_steps = graph_steps;
    }
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    CUDA_OK(cudaEventRecord(e0, st));
    int launched = 0;
    for (;;) {
        if (use_graph) {
            CUDA_OK(cudaGraphLaunch(s->graph, st));
            launched += graph_steps;
        } else {
            for (int i = 0; i < graph_steps; ++i) device_step(s, st);
            launched += graph_steps;
        }
        CUDA_OK(cudaMemcpyAsync(s->h_flag, s->n_active, 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaMemcpyAsync(s->h_flag + 1, s->step, 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
        if (s->h_flag[0] == 0 || launched > s->max_steps + graph_steps) break;
    }
    CUDA_OK(cudaEventRecord(e1, st));
    CUDA_OK(cudaEventSynchronize(e1));
    float ms = 0.0f;
    CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (gpu_ms) *gpu_ms = ms;
    int32_t flag = 0, cap_err = 0;
    CUDA_OK(cudaMemcpy(&flag, s->cache->ws.d_flag, 4, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(&cap_err, s->scalars + 4, 4, cudaMemcpyDeviceToHost));
    SD_CHECK(flag == 0, INTERNAL, "non-finite logit produced");
    SD_CHECK(cap_err == 0, CAPACITY, "padded grid outgrew the cache capacity during the device loop");
    return s->h_flag[1];
}

// Host-driven loop over the C-ABI verify step (the reference's loop shape:
// predictor on the host, H2D drafts, D2H tau + accepted every step).
int session_run_host(sd_session* s, float* gpu_ms, int64_t* h2d_bytes, int64_t* d2h_bytes) {
    SD_CHECK(s->prefilled, CONTRACT, "session has not been prefilled");
    SD_CHECK(s->e.predictor != 0, CONFIG, "the host-driven loop runs the retrieval / synthetic predictors");
    SD_CHECK(s->e.mode <= 2, CONFIG, "the ablation modes run in the device-resident loop only");
    cudaStream_t st = s->model->st;
    set_device(s->model->m.device);
    const int B = s->B;
    std::vector<std::vector<int32_t>> ctx(B);
    std::vector<int32_t> traj;
    if (s->e.predictor == 2) {
        SD_CHECK(s->traj, CONTRACT, "synthetic predictor needs a trajectory");
        traj.resize((size_t)B * s->traj_stride);
        CUDA_OK(cudaMemcpy(traj.data(), s->traj, 4 * traj.size(), cudaMemcpyDeviceToHost));
    }
    std::vector<int32_t> gen(B, s->e.max_new_tokens > 0 ? 1 : 0), active = s->snap_active, last(B), counts(B), budget(B), tau(B), clipped(B), acc,
        drafts;
    for (int b = 0; b < B; ++b) {
        ctx[b] = s->prompts[b];
        if (s->e.max_new_tokens > 0) ctx[b].push_back(s->first_tok[b]);
    }
    int64_t h2d = 0, d2h = 0;
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    CUDA_OK(cudaEventRecord(e0, st));
    int steps = 0;
    for (;; ++steps) {
        int nact = 0;
        for (int b = 0; b < B; ++b) nact += active[b];
        if (!nact) break;
        drafts.clear();
        int kmax = 0;
        for (int b = 0; b < B; ++b) {
            counts[b] = 0;
            if (!active[b]) continue;
            std::vector<int32_t> d;
            if (s->e.predictor == 1) {
                d = retrieval_predict(ctx[b], s->e.match_len, s->e.copy_len);
            } else {  // predictors.cpp:61-72 over the greedy continuation
                uint64_t rs = s->e.seed ^ ((uint64_t)steps * 0xD1B54A32D192ED03ULL) ^
                              ((uint64_t)(s->e.sample_id_base + b) * 0x8CB92BA72F3D8DD7ULL);  // global id
                auto nx = [&]() {
                    uint64_t z = (rs += 0x9E3779B97F4A7C15ULL);
                    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
                    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
                    return z ^ (z >> 31);
                };
                rs = nx();
                for (int i = 0; i < s->e.k; ++i) {
                    int t = traj[(size_t)b * s->traj_stride + gen[b] + i];
                    if ((double)(nx() >> 11) * 0x1.0p-53 >= s->e.synthetic_accuracy)
                        t = (t + 1) % s->model->m.cfg.vocab_size;
                    d.push_back(t);
                }
            }
            counts[b] = (int)d.size();
            kmax = std::max(kmax, counts[b]);
            drafts.insert(drafts.end(), d.begin(), d.end());
            last[b] = ctx[b].back();
            budget[b] = s->e.max_new_tokens - gen[b];
        }
        acc.assign((size_t)B * (kmax + 1), -1);
        verify_step_host(s->model, s->cache.get(), last.data(), counts.data(), drafts.data(), budget.data(),
                         active.data(), s->e.stop_on_eos, tau.data(), acc.data(), clipped.data(), nullptr);
        h2d += 4 * (4 * (int64_t)B + (int64_t)drafts.size()) + 8 * (int64_t)B;  // inputs + cache descriptors
        d2h += 4 * (2 * (int64_t)B + (int64_t)B * (s->kcap + 1)) + 4;
        for (int b = 0; b < B; ++b) {
            if (!active[b]) continue;
            for (int j = 0; j < tau[b]; ++j) ctx[b].push_back(acc[(size_t)b * (kmax + 1) + j]);
            gen[b] += tau[b];
            if (gen[b] >= s->e.max_new_tokens || (s->e.stop_on_eos && ctx[b].back() == 1)) active[b] = 0;
        }
    }
    CUDA_OK(cudaEventRecord(e1, st));
    CUDA_OK(cudaEventSynchronize(e1));
    float ms = 0.0f;
    CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (gpu_ms) *gpu_ms = ms;
    if (h2d_bytes) *h2d_bytes = h2d;
    if (d2h_bytes) *d2h_bytes = d2h;
    // leave the device-side session state consistent with what was generated
    std::vector<int32_t> len(B);
    for (int b = 0; b < B; ++b) {
        len[b] = (int)ctx[b].size();
        CUDA_OK(cudaMemcpy(s->ctx + (size_t)b * s->ctx_cap, ctx[b].data(), 4 * ctx[b].size(), cudaMemcpyHostToDevice));
    }
    CUDA_OK(cudaMemcpy(s->ctx_len, len.data(), 4 * (size_t)B, cudaMemcpyHostToDevice));
    return steps;
}

}  // namespace sdb

using namespace sdb;

namespace {
thread_local std::string g_serr;
template <class F>
int sguard(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_serr = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_serr = e.what();
        return INTERNAL;
    }
}
}  // namespace

extern "C" {

const char* sd_session_last_error(void) { return g_serr.c_str(); }

int sd_session_create(sd_model* m, const sd_engine_config* cfg, int capacity, sd_session** out) {
    return sguard([&] { *out = session_create(m, *cfg, capacity); });
}
int sd_session_create_draft(sd_model* target, sd_model* draft, const sd_engine_config* cfg, int capacity,
                            sd_session** out) {
    return sguard([&] { *out = session_create(target, *cfg, capacity, draft); });
}
int sd_session_prefill(sd_session* s, const int32_t* prompts, const int32_t* lens) {
    return sguard([&] { session_prefill(s, prompts, lens); });
}
int sd_session_set_trajectory(sd_session* s, const int32_t* traj, int stride) {
    return sguard([&] { session_set_trajectory(s, traj, stride); });
}
int sd_session_reset(sd_session* s) {
    return sguard([&] { session_reset(s); });
}
int sd_session_run(sd_session* s, int use_graph, int graph_steps, int32_t* steps, float* gpu_ms) {
    return sguard([&] { *steps = session_run(s, use_graph, graph_steps, gpu_ms); });
}
// n eager device steps (no graph, no completion check): profiling hook
int sd_session_step(sd_session* s, int n) {
    return sguard([&] {
        SD_CHECK(s->prefilled, CONTRACT, "session has not been prefilled");
        set_device(s->model->m.device);
        prepare_fast_kernels();
        for (int i = 0; i < n; ++i) device_step(s, s->model->st);
        CUDA_OK(cudaStreamSynchronize(s->model->st));
    });
}
int sd_session_run_host(sd_session* s, int32_t* steps, float* gpu_ms, int64_t* h2d_bytes, int64_t* d2h_bytes) {
    return sguard([&] { *steps = session_run_host(s, gpu_ms, h2d_bytes, d2h_bytes); });
}
int sd_session_outputs(sd_session* s, int32_t* gen_tokens, int32_t* gen_counts, int32_t* log_k, int32_t* log_tau,
                       int max_steps) {
    return sguard([&] {
        int B = s->B, mx = s->e.max_new_tokens;
        std::vector<int32_t> len(B), ctx((size_t)B * s->ctx_cap);
        CUDA_OK(cudaMemcpy(len.data(), s->ctx_len, 4 * (size_t)B, cudaMemcpyDeviceToHost));
        CUDA_OK(cudaMemcpy(ctx.data(), s->ctx, 4 * ctx.size(), cudaMemcpyDeviceToHost));
        for (int b = 0; b < B; ++b) {
            int g = len[b] - s->prompt_lens[b];
            gen_counts[b] = g;
            std::memcpy(gen_tokens + (size_t)b * mx, ctx.data() + (size_t)b * s->ctx_cap + s->prompt_lens[b],
                        4 * (size_t)std::min(g, mx));
        }
        int n = std::min(max_steps, s->max_steps);
        if (log_k) CUDA_OK(cudaMemcpy(log_k, s->log_k, 4 * (size_t)n * B, cudaMemcpyDeviceToHost));
        if (log_tau) CUDA_OK(cudaMemcpy(log_tau, s->log_tau, 4 * (size_t)n * B, cudaMemcpyDeviceToHost));
    });
}
int sd_session_draft_log(sd_session* s, int32_t* drafts, int max_steps) {
    return sguard([&] {
        int n = std::min(max_steps, s->max_steps);
        CUDA_OK(cudaMemcpy(drafts, s->log_drafts, 4 * (size_t)n * s->B * std::max(1, s->kcap),
                           cudaMemcpyDeviceToHost));
    });
}
int sd_session_gather_outputs(sd_session* s, sd_comm* comm, int32_t* gen_tokens, int32_t* gen_counts) {
    return sguard([&] {
        const int B = s->B, mx = s->e.max_new_tokens;
        // one int32 block per rank: [B][max_new] tokens then [B] counts
        std::vector<int32_t> mine((size_t)B * mx + B);
        CUDA_OK(cudaSetDevice(s->model->m.device));
        if (sd_session_outputs(s, mine.data(), mine.data() + (size_t)B * mx, nullptr, nullptr, 0) != 0)
            throw Error(INTERNAL, "session outputs unavailable");
        int world = 0, rank = 0;
        if (sd_comm_size(comm, &world, &rank) != 0) throw Error(INTERNAL, sd_comm_last_error());
        std::vector<int32_t> all(mine.size() * (size_t)world);
        if (sd_comm_allgather_i32(comm, mine.data(), (int64_t)mine.size(), all.data()) != 0)
            throw Error(INTERNAL, sd_comm_last_error());
        for (int r = 0; r < world; ++r) {
            const int32_t* blk = all.data() + (size_t)r * mine.size();
            std::memcpy(gen_tokens + (size_t)r * B * mx, blk, 4 * (size_t)B * mx);
            std::memcpy(gen_counts + (size_t)r * B, blk + (size_t)B * mx, 4 * (size_t)B);
        }
    });
}
int sd_session_cache(sd_session* s, sd_cache** out) {
    return sguard([&] { *out = s->cache.get(); });
}
void sd_session_destroy(sd_session* s) {
    if (s) {
        cudaSetDevice(s->model->m.device);
        delete s;
    }
}

}  // extern "C"
