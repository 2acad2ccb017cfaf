// Device kernels of one verify step that surround the forward pass:
//   k_predict    drafts on device for the resident loop: LLMA prompt lookup
//                (predictors.cpp:39-59) or the synthetic corrupted greedy
//                rollout (predictors.cpp:61-72, engine.cpp:182-185)
//   k_pack       Algorithm 1 (ragged.cpp:6-17) + the slot/plan construction of
//                engine.cpp:427-444 (EMS) or 408-426 (vanilla), plus the
//                per-sample ragged descriptors the attention kernel reads
//   k_accept     greedy verification (engine.cpp:60-76), budget/EOS clipping
//                (engine.cpp:454-475) and the per-sample commit
//                (kv_cache.cpp:152-161; padded: 269-314 metadata)
//   k_pad_fill   the vanilla layout's zero filler rows (kv_cache.cpp:295-307)
#include <cuda_bf16.h>

#include <climits>

#include "common.h"
#include "pdl.cuh"
#include "step.h"
#include "trace.cuh"

SD_TRACE_TU(step)

namespace sdb {

__device__ __forceinline__ int32_t last_token(const StepArgs& a, int s) {
    return a.last ? a.last[s] : a.ctx[(size_t)s * a.ctx_cap + a.ctx_len[s] - 1];
}
__device__ __forceinline__ int32_t draft_at(const StepArgs& a, int s, int doff, int j) {
    return a.draft_stride ? a.drafts[(size_t)s * a.draft_stride + j] : a.drafts[doff + j];
}

// Block-wide reductions / exclusive scan over one value per thread (256
// threads): warp shuffles, then the 8 warp results through shared memory.
constexpr int kStepThreads = 256;
__device__ __forceinline__ int block_reduce_max(int v, int* sw) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = __reduce_max_sync(0xffffffffu, v);
    if (lane == 0) sw[warp] = v;
    __syncthreads();
    int r = sw[0];
#pragma unroll
    for (int w = 1; w < kStepThreads / 32; ++w) r = max(r, sw[w]);
    __syncthreads();
    return r;
}
__device__ __forceinline__ int block_reduce_min(int v, int* sw) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = __reduce_min_sync(0xffffffffu, v);
    if (lane == 0) sw[warp] = v;
    __syncthreads();
    int r = sw[0];
#pragma unroll
    for (int w = 1; w < kStepThreads / 32; ++w) r = min(r, sw[w]);
    __syncthreads();
    return r;
}
// exclusive prefix sums of two values at once; `tot` receives the block totals
__device__ __forceinline__ int2 block_excl_scan2(int2 v, int2* sw, int2& tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int2 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int yx = __shfl_up_sync(0xffffffffu, x.x, o), yy = __shfl_up_sync(0xffffffffu, x.y, o);
        if (lane >= o) {
            x.x += yx;
            x.y += yy;
        }
    }
    if (lane == 31) sw[warp] = x;
    __syncthreads();
    int2 off = make_int2(0, 0);
    tot = make_int2(0, 0);
#pragma unroll
    for (int w = 0; w < kStepThreads / 32; ++w) {
        if (w < warp) {
            off.x += sw[w].x;
            off.y += sw[w].y;
        }
        tot.x += sw[w].x;
        tot.y += sw[w].y;
    }
    __syncthreads();
    return make_int2(off.x + x.x - v.x, off.y + x.y - v.y);
}

// One block of 256 threads.  The prefix sums of Algorithm 1 (ragged.cpp:6-17)
// run as block scans over the samples (no serial per-sample loop), then every
// thread fills the token / plan rows of its samples.
__global__ void __launch_bounds__(kStepThreads) k_pack(StepArgs a) {
    CtaTrace trace__(TK_PACK);
    pdl_trigger();
    pdl_wait();
    __shared__ int s_red[kStepThreads / 32];
    __shared__ int2 s_scan[kStepThreads / 32];
    const int B = a.B;
    // padded input rows (1 + k_max per sample)?  The layout's own choice unless
    // an ablation mode decouples input padding from KV padding.
    const bool pad_in = a.layout == PADDED ? a.ablation != 1 : a.ablation == 2;
    int km = 0, first = INT_MAX;
    for (int s = threadIdx.x; s < B; s += kStepThreads)
        if (a.active[s]) {
            km = max(km, a.counts[s]);
            first = min(first, s);
        }
    const int kmax = block_reduce_max(km, s_red);
    first = block_reduce_min(first, s_red);
    const int base = a.layout == PADDED && first < B ? a.committed[first] : -1;
    // draft_off / first_row: exclusive prefix sums over the active samples
    int2 carry = make_int2(0, 0);  // (drafts, rows) before this chunk of samples
    bool over = false;
    for (int c0 = 0; c0 < B; c0 += kStepThreads) {
        const int s = c0 + threadIdx.x;
        const bool act = s < B && a.active[s];
        const int ks = act ? a.counts[s] : 0;
        int2 tot;
        const int2 ex = block_excl_scan2(make_int2(ks, act ? 1 + (pad_in ? kmax : ks) : 0), s_scan, tot);
        if (s < B) {
            a.draft_off[s] = carry.x + ex.x;
            a.first_row[s] = carry.y + ex.y;
        }
        // Capacity guard for the device-resident loop (the host-driven step
        // checks on the host first): never write past a sample's extent.
        if (act) {
            const int last = a.layout == PADDED ? base + kmax : a.committed[s] + (pad_in ? kmax : ks);
            if (last >= a.cap) over = true;
        }
        carry.x += tot.x;
        carry.y += tot.y;
    }
    over = __syncthreads_or(over);
    if (over)
        for (int s = threadIdx.x; s < B; s += kStepThreads) a.active[s] = 0;
    if (threadIdx.x == 0) {
        if (over) a.scalars[4] = 2;       // CapacityError, reported by the host
        a.scalars[0] = over ? 0 : carry.y;  // T
        a.scalars[1] = kmax;              // k_max
        a.scalars[2] = base;              // padded grid base row
    }
    __syncthreads();  // active flags cleared on overflow
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        const int row0 = a.first_row[s];
        if (!a.active[s]) {
            a.segs[s] = SampleSeg{row0, 0, 0, 0};
            continue;
        }
        int ks = a.counts[s], d0 = a.draft_off[s];
        int n = pad_in ? 1 + kmax : 1 + ks;
        int kv_len = 0;
        if (a.layout == PADDED && !pad_in)  // unpadded input over the grid: the alignment rows are holes
            for (int o = 1 + ks; o <= kmax; ++o) a.pad[(size_t)s * a.cap + base + o] = 1;
        for (int o = 0; o < n; ++o) {
            bool real = o <= ks;
            int tok = o == 0 ? last_token(a, s) : (real ? draft_at(a, s, d0, o - 1) : 2 /* tok::kPad */);
            Plan p;
            p.sample = s;
            if (a.layout == PADDED) {
                p.logical_pos = a.logical[s] + o;
                p.write_slot = base + o;
                p.store = real ? 1 : 0;
                a.pad[(size_t)s * a.cap + base + o] = real ? 0 : 1;  // write_kv / mark_hole
            } else {
                p.logical_pos = a.committed[s] + o;
                p.write_slot = p.logical_pos;
                p.store = real ? 1 : 0;  // PAD spectators (ablation 2) store nothing
            }
            a.tokens[row0 + o] = tok;
            a.plans[row0 + o] = p;
            a.qidx[row0 + o] = row0 + o;
            kv_len = p.write_slot + 1;
        }
        a.segs[s] = SampleSeg{row0, n, kv_len, 0};
    }
}

// One block, one thread per sample.
__global__ void k_accept(StepArgs a) {
    CtaTrace trace__(TK_ACCEPT);
    pdl_trigger();
    pdl_wait();
    __shared__ int s_taumax, s_active, s_step;
    if (threadIdx.x == 0) {
        s_taumax = 0;
        s_active = 0;
        s_step = a.step ? *a.step : 0;
    }
    __syncthreads();
    const int B = a.B, W = a.acc_stride;
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        const bool logging = a.log_tau && s_step < a.max_steps;
        if (!a.active[s]) {
            a.tau[s] = 0;
            a.clipped[s] = 0;
            if (logging) {
                a.log_tau[(size_t)s_step * B + s] = 0;
                a.log_k[(size_t)s_step * B + s] = -1;
            }
            continue;
        }
        int ks = a.counts[s], row0 = a.first_row[s], d0 = a.draft_off[s];
        int vt = ks + 1;
        // picks and drafts of up to kAccBatch positions loaded before the
        // first comparison (one round trip instead of one per position); the
        // verification itself is the reference's first-mismatch scan
        constexpr int kAccBatch = 16;
        int pick[kAccBatch], drf[kAccBatch];
#pragma unroll
        for (int j = 0; j < kAccBatch; ++j) {
            pick[j] = j <= ks ? a.argmax[row0 + j] : 0;
            drf[j] = j < ks ? draft_at(a, s, d0, j) : -1;
        }
        bool hit = false;
#pragma unroll
        for (int j = 0; j < kAccBatch; ++j) {
            if (hit || j > ks) break;
            a.accepted[s * W + j] = pick[j];
            if (j < ks && pick[j] != drf[j]) {
                vt = j + 1;
                hit = true;
            }
        }
        for (int j = kAccBatch; !hit && j <= ks; ++j) {  // k > 15 only
            int x = a.argmax[row0 + j];
            a.accepted[s * W + j] = x;
            if (j < ks && x != draft_at(a, s, d0, j)) {
                vt = j + 1;
                hit = true;
            }
        }
        int budget = a.budget ? a.budget[s] : a.max_new - a.gen[s];
        int tau = vt < budget ? vt : budget;
        if (a.stop_on_eos) {  // first EOS among the accepted tokens ends the sample
            int eos = -1;
#pragma unroll
            for (int j = 0; j < kAccBatch; ++j)
                if (eos < 0 && j < tau && pick[j] == 1 /* tok::kEos */) eos = j;
            for (int j = kAccBatch; eos < 0 && j < tau; ++j)
                if (a.accepted[s * W + j] == 1) eos = j;
            if (eos >= 0) tau = eos + 1;
        }
        a.tau[s] = tau;
        a.clipped[s] = tau < vt ? 1 : 0;
        atomicMax(&s_taumax, tau);
        if (a.layout == UNPAD) a.committed[s] += tau;  // kv_cache.cpp:158
        if (a.ctx) {  // device-resident loop: append, advance, finish (engine.cpp:465-470)
            int len = a.ctx_len[s];
            int last_tok = 0;
            int32_t* cp = a.ctx + (size_t)s * a.ctx_cap + len;
#pragma unroll
            for (int j = 0; j < kAccBatch; ++j)
                if (j < tau) {
                    cp[j] = pick[j];
                    last_tok = pick[j];
                }
            for (int j = kAccBatch; j < tau; ++j) {
                last_tok = a.accepted[s * W + j];
                cp[j] = last_tok;
            }
            a.ctx_len[s] = len + tau;
            int g = a.gen[s] + tau;
            a.gen[s] = g;
            bool done = g >= a.max_new || (a.stop_on_eos && last_tok == 1);
            if (done) a.active[s] = 0;
            else atomicAdd(&s_active, 1);
        }
        if (logging) {
            a.log_tau[(size_t)s_step * B + s] = tau + (a.clipped[s] ? 0x10000 : 0);
            a.log_k[(size_t)s_step * B + s] = ks;
            if (a.log_drafts)
                for (int j = 0; j < ks && j < a.log_kcap; ++j)
                    a.log_drafts[((size_t)s_step * B + s) * a.log_kcap + j] = draft_at(a, s, d0, j);
        }
    }
    __syncthreads();
    if (a.layout == PADDED) {
        int tmax = s_taumax;
        if (threadIdx.x == 0) a.scalars[3] = tmax;
        for (int s = threadIdx.x; s < B; s += blockDim.x) {
            if (!a.tau[s]) continue;
            int base = a.committed[s];
            for (int r = base + a.tau[s]; r < base + tmax; ++r) a.pad[(size_t)s * a.cap + r] = 1;
            a.committed[s] = base + tmax;  // kv_cache.cpp:309
            a.logical[s] += a.tau[s];      // kv_cache.cpp:310
        }
    }
    if (threadIdx.x == 0) {
        if (a.n_active) *a.n_active = s_active;
        // count only steps that verified something (graph replays may run
        // trailing no-op steps after every sample finished)
        if (a.step && s_taumax > 0) *a.step = s_step + 1;
        if (a.has_cond)  // keep looping while a sample is active (and the step log has room)
            cudaGraphSetConditional((cudaGraphConditionalHandle)a.cond,
                                    (s_active > 0 && s_step + 1 < a.max_steps) ? 1u : 0u);
    }
}

// Zero K/V filler rows [base + tau_s, base + tau_max) for every layer
// (kv_cache.cpp:295-307).  Runs after k_accept, so committed is already
// base + tau_max.  grid = (L * 2, B), block 256.
template <typename T>
__global__ void k_pad_fill(StepArgs a, T* kv, int heads, int hd) {
    CtaTrace trace__(TK_PAD_FILL);
    pdl_trigger();
    pdl_wait();
    int lw = blockIdx.x, s = blockIdx.y;
    if (!a.tau[s]) return;
    int tmax = a.scalars[3];
    int end = a.committed[s], base = end - tmax;
    int r0 = base + a.tau[s];
    int rows = end - r0;
    if (rows <= 0) return;
    for (int head = 0; head < heads; ++head) {
        T* p = kv + (((size_t)lw * a.B + s) * heads + head) * (size_t)a.cap * hd + (size_t)r0 * hd;
        for (int i = threadIdx.x; i < rows * hd; i += blockDim.x) p[i] = T(0.0f);
    }
}

// grid = (L * 2, n), block 256: zero rows [r0[i], r1) of sample samples[i]
template <typename T>
__global__ void k_zero_rows(T* kv, const int32_t* samples, const int32_t* r0, int r1, int B, int heads, int cap,
                            int hd) {
    CtaTrace trace__(TK_PAD_FILL);
    pdl_trigger();
    pdl_wait();
    const int lw = blockIdx.x, s = samples[blockIdx.y], a = r0[blockIdx.y];
    const int rows = r1 - a;
    if (rows <= 0) return;
    for (int head = 0; head < heads; ++head) {
        T* p = kv + (((size_t)lw * B + s) * heads + head) * (size_t)cap * hd + (size_t)a * hd;
        for (int i = threadIdx.x; i < rows * hd; i += blockDim.x) p[i] = T(0.0f);
    }
}

__device__ __forceinline__ uint64_t splitmix_next(uint64_t& st) {  // rng.hpp:15-20
    uint64_t z = (st += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// grid = B, block 128
__global__ void k_predict(StepArgs a, PredictArgs p) {
    CtaTrace trace__(TK_PREDICT);
    pdl_trigger();
    pdl_wait();
    const int s = blockIdx.x;
    __shared__ int s_best;
    if (!a.active[s]) {
        if (threadIdx.x == 0) a.counts[s] = 0;
        return;
    }
    const int32_t* ctx = a.ctx + (size_t)s * a.ctx_cap;
    int32_t* out = a.drafts + (size_t)s * a.draft_stride;
    if (p.kind == 1) {  // predictors.cpp:39-59: rightmost earlier match of the trailing n-gram
        const int len = a.ctx_len[s], suffix = len - p.match_len;
        if (threadIdx.x == 0) s_best = -1;
        __syncthreads();
        if (suffix > 0) {
            for (int start = suffix - 1 - threadIdx.x; start >= 0; start -= blockDim.x) {
                bool ok = true;
                for (int i = 0; i < p.match_len && ok; ++i) ok = ctx[start + i] == ctx[suffix + i];
                if (ok) {
                    atomicMax(&s_best, start);
                    break;  // later candidates of this thread are further left
                }
            }
        }
        __syncthreads();
        int best = s_best;
        int take = 0;
        if (best >= 0) {
            int from = best + p.match_len;
            take = min(p.copy_len, len - from);
            for (int i = threadIdx.x; i < take; i += blockDim.x) out[i] = ctx[from + i];
        }
        if (threadIdx.x == 0) a.counts[s] = take;
    } else {  // predictors.cpp:61-72 over the precomputed greedy continuation
        if (threadIdx.x == 0) {
            int g = a.gen[s];
            uint64_t st = p.seed ^ ((uint64_t)(*a.step) * 0xD1B54A32D192ED03ULL) ^
                          ((uint64_t)(p.id_base + s) * 0x8CB92BA72F3D8DD7ULL);  // mix_seed (rng.hpp:43-46), global id
            st = splitmix_next(st);
            for (int i = 0; i < p.k; ++i) {
                int t = p.traj[(size_t)s * p.traj_stride + g + i];
                double u = (double)(splitmix_next(st) >> 11) * 0x1.0p-53;
                if (u >= p.accuracy) t = (t + 1) % p.vocab;
                out[i] = t;
            }
            a.counts[s] = p.k;
        }
    }
}

// Draft step j's ragged batch: j == 0 feeds the context tokens the draft
// cache lacks (1 after a rejection, 2 when every draft was accepted plus the
// bonus token), j > 0 feeds draft j-1.  One block.
__global__ void k_draft_pack(DraftArgs d, int j) {
    CtaTrace trace__(TK_DRAFT_PACK);
    pdl_trigger();
    pdl_wait();
    __shared__ int s_row0[256 + 1];
    const int B = d.B;
    if (threadIdx.x == 0) {
        int t = 0;
        for (int s = 0; s < B; ++s) {
            s_row0[s] = t;
            if (d.active[s]) t += j == 0 ? d.ctx_len[s] - d.dcommit[s] : 1;
        }
        s_row0[B] = t;
        *d.dT = t;
    }
    __syncthreads();
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        const int row0 = s_row0[s], n = s_row0[s + 1] - row0;
        if (n == 0) {
            d.segs[s] = SampleSeg{row0, 0, 0, 0};
            continue;
        }
        if (j == 0) d.lsnap[s] = d.ctx_len[s];
        const int pos0 = j == 0 ? d.dcommit[s] : d.ctx_len[s] + j - 1;
        for (int o = 0; o < n; ++o) {
            const int pos = pos0 + o;
            d.tokens[row0 + o] = j == 0 ? d.ctx[(size_t)s * d.ctx_cap + pos] : d.drafts[(size_t)s * d.kcap + j - 1];
            d.plans[row0 + o] = Plan{s, pos, pos, 1};
            d.qidx[row0 + o] = row0 + o;
        }
        d.segs[s] = SampleSeg{row0, n, pos0 + n, 0};
    }
}

// draft j = greedy_next of the sample's last row (model.cpp:34-41)
__global__ void k_draft_take(DraftArgs d, int j) {
    CtaTrace trace__(TK_DRAFT_TAKE);
    pdl_trigger();
    pdl_wait();
    for (int s = threadIdx.x; s < d.B; s += blockDim.x) {
        if (!d.active[s]) {
            d.counts[s] = 0;
            continue;
        }
        const SampleSeg g = d.segs[s];
        d.drafts[(size_t)s * d.kcap + j] = d.argmax[g.q_start + g.n_q - 1];
        d.counts[s] = j + 1;
        if (j == 0) d.dcommit[s] = d.lsnap[s];  // every context token is in the draft cache
    }
}

// After verification: the draft KV of positions lsnap .. lsnap+tau-2 holds the
// accepted x_0..x_{tau-2} (= the drafts), so it stays; the rest is forgotten
// (rollback by metadata, as UnpadArena::commit_accepted, kv_cache.cpp:158).
__global__ void k_draft_commit(DraftArgs d) {
    CtaTrace trace__(TK_DRAFT_COMMIT);
    pdl_trigger();
    pdl_wait();
    for (int s = threadIdx.x; s < d.B; s += blockDim.x) {
        const int tau = d.tau[s];
        if (tau > 0) d.dcommit[s] = d.lsnap[s] + min(tau - 1, d.k - 1);
    }
}

void launch_draft_pack(const DraftArgs& d, int j, cudaStream_t st) {
    launch_k(k_draft_pack, dim3(1), dim3(256), 0, st, d, j);
}
void launch_draft_take(const DraftArgs& d, int j, cudaStream_t st) {
    launch_k(k_draft_take, dim3(1), dim3(256), 0, st, d, j);
}
void launch_draft_commit(const DraftArgs& d, cudaStream_t st) { launch_k(k_draft_commit, dim3(1), dim3(256), 0, st, d); }

void launch_pack(const StepArgs& a, cudaStream_t st) { launch_k(k_pack, dim3(1), dim3(kStepThreads), 0, st, a); }
void launch_accept(const StepArgs& a, cudaStream_t st) { launch_k(k_accept, dim3(1), dim3(256), 0, st, a); }
void launch_pad_fill(const StepArgs& a, const Cache& c, cudaStream_t st) {
    dim3 grid(c.L * 2, c.B);
    if (c.elem_bytes == 4)
        launch_k(k_pad_fill<float>, grid, dim3(256), 0, st, a, (float*)c.kv, c.heads, c.hd);
    else
        launch_k(k_pad_fill<__nv_bfloat16>, grid, dim3(256), 0, st, a, (__nv_bfloat16*)c.kv, c.heads, c.hd);
}
void launch_zero_rows(const Cache& c, const int32_t* samples, const int32_t* r0, int n, int r1, cudaStream_t st) {
    dim3 grid(c.L * 2, n);
    if (c.elem_bytes == 4)
        launch_k(k_zero_rows<float>, grid, dim3(256), 0, st, (float*)c.kv, samples, r0, r1, c.B, c.heads, c.cap, c.hd);
    else
        launch_k(k_zero_rows<__nv_bfloat16>, grid, dim3(256), 0, st, (__nv_bfloat16*)c.kv, samples, r0, r1, c.B,
                 c.heads, c.cap, c.hd);
}
void launch_predict(const StepArgs& a, const PredictArgs& p, cudaStream_t st) {
    launch_k(k_predict, dim3(a.B), dim3(128), 0, st, a, p);
}

}  // namespace sdb
