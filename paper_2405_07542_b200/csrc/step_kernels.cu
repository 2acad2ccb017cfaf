// Device kernels of one verify step that surround the forward pass:
//   k_pack       Algorithm 1 (ragged.cpp:6-17) + the slot/plan construction of
//                engine.cpp:427-444 (EMS) or 408-426 (vanilla) on device
//   k_accept     greedy verification (engine.cpp:60-76), budget/EOS clipping
//                (engine.cpp:454-463) and the per-sample commit
//                (kv_cache.cpp:152-161; padded: 269-314 metadata)
//   k_pad_fill   the vanilla layout's zero filler rows (kv_cache.cpp:295-307)
#include <cuda_bf16.h>

#include "common.h"
#include "step.h"

namespace sdb {

// One block.  Thread 0 runs the O(B) prefix sums (B <= a few hundred), then
// every thread fills token/plan rows in parallel.
__global__ void k_pack(StepArgs a) {
    const int B = a.B;
    if (threadIdx.x == 0) {
        int t = 0, d = 0, kmax = 0;
        for (int s = 0; s < B; ++s)
            if (a.active[s] && a.counts[s] > kmax) kmax = a.counts[s];
        int base = -1;
        for (int s = 0; s < B; ++s) {
            a.draft_off[s] = d;
            d += a.counts[s];
            a.first_row[s] = t;
            if (!a.active[s]) continue;
            if (a.layout == PADDED) {
                if (base < 0) base = a.committed[s];
                t += 1 + kmax;
            } else {
                t += 1 + a.counts[s];
            }
        }
        a.scalars[0] = t;     // T
        a.scalars[1] = kmax;  // k_max
        a.scalars[2] = base;  // padded grid base row
    }
    __syncthreads();
    const int kmax = a.scalars[1], base = a.scalars[2];
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        if (!a.active[s]) continue;
        int ks = a.counts[s], row0 = a.first_row[s], d0 = a.draft_off[s];
        int n = a.layout == PADDED ? 1 + kmax : 1 + ks;
        for (int o = 0; o < n; ++o) {
            bool real = o <= ks;
            int tok = o == 0 ? a.last[s] : (real ? a.drafts[d0 + o - 1] : 2 /* tok::kPad */);
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
                p.store = 1;
            }
            a.tokens[row0 + o] = tok;
            a.plans[row0 + o] = p;
        }
    }
}

// One block, one thread per sample.
__global__ void k_accept(StepArgs a) {
    __shared__ int s_taumax;
    if (threadIdx.x == 0) s_taumax = 0;
    __syncthreads();
    const int B = a.B, W = a.acc_stride;
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        if (!a.active[s]) {
            a.tau[s] = 0;
            a.clipped[s] = 0;
            continue;
        }
        int ks = a.counts[s], row0 = a.first_row[s], d0 = a.draft_off[s];
        int vt = ks + 1;
        for (int j = 0; j <= ks; ++j) {
            int x = a.argmax[row0 + j];
            a.accepted[s * W + j] = x;
            if (j < ks && x != a.drafts[d0 + j]) {
                vt = j + 1;
                break;
            }
        }
        int tau = vt < a.budget[s] ? vt : a.budget[s];
        if (a.stop_on_eos) {
            for (int j = 0; j < tau; ++j) {
                if (a.accepted[s * W + j] == 1 /* tok::kEos */) {
                    tau = j + 1;
                    break;
                }
            }
        }
        a.tau[s] = tau;
        a.clipped[s] = tau < vt ? 1 : 0;
        atomicMax(&s_taumax, tau);
        if (a.layout == UNPAD) a.committed[s] += tau;  // kv_cache.cpp:158
    }
    __syncthreads();
    if (a.layout == PADDED) {
        int tmax = s_taumax;
        if (threadIdx.x == 0) a.scalars[3] = tmax;
        for (int s = threadIdx.x; s < B; s += blockDim.x) {
            if (!a.active[s]) continue;
            int base = a.committed[s];
            for (int r = base + a.tau[s]; r < base + tmax; ++r) a.pad[(size_t)s * a.cap + r] = 1;
            a.committed[s] = base + tmax;  // kv_cache.cpp:309
            a.logical[s] += a.tau[s];      // kv_cache.cpp:310
        }
    }
}

// Zero K/V filler rows [base + tau_s, base + tau_max) for every layer
// (kv_cache.cpp:295-307).  Runs after k_accept, so committed is already
// base + tau_max.  grid = (L * 2, B), block 256.
template <typename T>
__global__ void k_pad_fill(StepArgs a, T* kv, int heads, int hd) {
    int lw = blockIdx.x, s = blockIdx.y;
    if (!a.active[s]) return;
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

void launch_pack(const StepArgs& a, cudaStream_t st) { k_pack<<<1, 256, 0, st>>>(a); }
void launch_accept(const StepArgs& a, cudaStream_t st) { k_accept<<<1, 256, 0, st>>>(a); }
void launch_pad_fill(const StepArgs& a, const Cache& c, cudaStream_t st) {
    dim3 grid(c.L * 2, c.B);
    if (c.elem_bytes == 4)
        k_pad_fill<float><<<grid, 256, 0, st>>>(a, (float*)c.kv, c.heads, c.hd);
    else
        k_pad_fill<__nv_bfloat16><<<grid, 256, 0, st>>>(a, (__nv_bfloat16*)c.kv, c.heads, c.hd);
}

}  // namespace sdb
