/* specdec_b200_debug.h — kernel-level test hooks (not part of the drop-in
 * boundary).  Used by tests/ to check the tcgen05 GEMM in isolation. */
#ifndef SPECDEC_B200_DEBUG_H
#define SPECDEC_B200_DEBUG_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* Y[T][M] = X[T][K] . W[M][K]^T with bf16 inputs (raw bits) and fp32 output,
 * through the stream-K tcgen05 kernel on `grid` CTAs (0 = one per SM).
 * Returns the kernel time in microseconds in *usec (CUDA events). */
/* flags bit 3: time the streaming kernel alone (no split-K reduction; Y untouched);
 * bit 7: time ten launches back to back (mean); bits 4-6 select bottleneck
 * probes (skip MMAs / token loads / partial stores) that only a probe build of
 * the kernel (-DSD_GEMM_PROBE, tools/gemm_probe.py --probe) honours */
int sd_debug_gemm(const uint16_t* W, const uint16_t* X, int M, int K, int T, int grid, int flags, float* Y,
                  float* usec);
/* In-graph kernel timeline (tools/timeline.py): while on, every CTA of every
 * verify-step kernel appends {kernel id, block, SM, grid size, t_entry, t_exit}
 * (globaltimer ns, 32 bytes) to a device buffer of `cap` records. */
int sd_debug_trace_begin(int cap);
/* The production persistent tcgen05 attention on caller-provided bf16
 * tensors of one layer:
 *   q [T][heads*hd]; kv [2][B][heads][cap][hd] (K then V); queries packed
 *   sample by sample, n_q[B] of them per sample, kv_len[B] visible extent,
 *   write_slot[T] per query (it sees keys <= its slot), pad [B][cap] flags or
 *   NULL -> ctx [T][heads*hd] bf16.  T <= 256.  *usec: one launch. */
int sd_debug_attention(const uint16_t* q, const uint16_t* kv, int B, int heads, int hd, int cap, const int32_t* n_q,
                       const int32_t* kv_len, const int32_t* write_slot, const uint8_t* pad, uint16_t* ctx,
                       float* usec);
int sd_debug_trace_end(void* out, int cap, int* n);
/* 1 if the bf16 model runs its layer GEMMs as cluster split-K launches with
 * fused reductions / LayerNorms (small models, gemm_cluster.cu), 0 if through
 * the stream-K GEMM + reduction kernels, negative on error.  SD_COMPACT=0 in
 * the environment when the model is created forces the stream-K path. */
struct sd_model;
int sd_debug_model_compact(const struct sd_model* m);
#ifdef __cplusplus
}
#endif
#endif
