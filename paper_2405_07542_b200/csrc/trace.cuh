// In-graph kernel timeline: every CTA of every verify-step kernel appends one
// record {kernel id, block, SM, %globaltimer at entry and at exit} to a
// device ring when tracing is on (a null buffer pointer otherwise: one load
// and a branch per CTA).  Unlike ncu, which serialises launches, this sees
// the real overlap of a PDL chain replayed from a CUDA graph, so the gaps
// between kernels and the SM occupancy of each phase can be measured.
//
// __device__ variables are per translation unit (no -rdc), so each .cu that
// traces declares its own buffer with SD_TRACE_TU and exports a setter.
#pragma once
#include <cstdint>

namespace sdb {

struct TraceRec {
    uint32_t kid, blk, smid, n;
    uint64_t t0, t1;
};

enum TraceKid : uint32_t {
    TK_GEMM = 1, TK_RED_STORE, TK_RED_GELU, TK_RED_QKV, TK_RED_RESID, TK_LN_ROWS, TK_ARGMAX,
    TK_EMBED_LN, TK_ATTN, TK_ATTN_COMBINE, TK_PREDICT, TK_PACK, TK_ACCEPT, TK_PAD_FILL,
    TK_DRAFT_PACK, TK_DRAFT_TAKE, TK_DRAFT_COMMIT, TK_GEMM_CL_QKV, TK_GEMM_CL_GELU, TK_GEMM_CL_RESID, TK_ATTN_WIDE,
    // trace points (kid >= 100): one record, tag = payload
    TK_ATTN_BYTES = 110,  // per attention CTA: algorithmic K/V bytes >> 10
};

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t s;
    asm volatile("mov.u32 %0, %smid;" : "=r"(s));
    return s;
}

struct TraceBuf {
    TraceRec* rec;
    unsigned* count;
    unsigned cap;
};

}  // namespace sdb

#define SD_TRACE_TU(name)                                                                 \
    namespace sdb {                                                                       \
    static __device__ TraceBuf g_trace_##name;                                            \
    void trace_set_##name(const TraceBuf& b) {                                            \
        CUDA_OK(cudaMemcpyToSymbol(g_trace_##name, &b, sizeof(b)));                       \
    }                                                                                     \
    namespace {                                                                           \
    [[maybe_unused]] __device__ __forceinline__ void trace_point(uint32_t kid, uint32_t tag) { \
        const TraceBuf& b = g_trace_##name;                                               \
        if (b.rec) {                                                                      \
            const uint64_t t = globaltimer(); /* before the (contended) slot atomic */   \
            unsigned i = atomicAdd(b.count, 1u);                                          \
            if (i < b.cap) b.rec[i] = TraceRec{kid, tag, smid(), 0, t, t};                \
        }                                                                                 \
    }                                                                                     \
    struct CtaTrace {                                                                     \
        uint64_t t0;                                                                      \
        TraceRec* rec; /* read once at entry: no global load on the exit path */          \
        uint32_t kid;                                                                     \
        __device__ __forceinline__ explicit CtaTrace(uint32_t k) : kid(k) {               \
            rec = g_trace_##name.rec;                                                     \
            t0 = rec ? globaltimer() : 0;                                                 \
        }                                                                                 \
        /* phase record from any thread (kid >= 100), free when tracing is off */         \
        template <int = 0> __device__ __forceinline__ void point(uint32_t pk, uint32_t tag) const { \
            if (rec) trace_point(pk, tag);                                                \
        }                                                                                 \
        __device__ __forceinline__ ~CtaTrace() {                                          \
            if (threadIdx.x == 0 && rec) {                                                \
                const TraceBuf& b = g_trace_##name;                                       \
                const uint64_t t1 = globaltimer();                                        \
                unsigned i = atomicAdd(b.count, 1u);                                      \
                if (i < b.cap) {                                                          \
                    uint32_t blk = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
                    b.rec[i] = TraceRec{kid, blk, smid(), gridDim.x * gridDim.y * gridDim.z, t0, t1}; \
                }                                                                         \
            }                                                                             \
        }                                                                                 \
    };                                                                                    \
    }                                                                                     \
    }
