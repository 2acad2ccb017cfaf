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
/* flags bit 0: store W tile-major ([m_tile][K/64][256][64], one contiguous 32 KB
 * TMA box per k-block) instead of row-major */
int sd_debug_gemm(const uint16_t* W, const uint16_t* X, int M, int K, int T, int grid, int flags, float* Y,
                  float* usec);
/* In-graph kernel timeline (tools/timeline.py): while on, every CTA of every
 * verify-step kernel appends {kernel id, block, SM, grid size, t_entry, t_exit}
 * (globaltimer ns, 32 bytes) to a device buffer of `cap` records. */
int sd_debug_trace_begin(int cap);
int sd_debug_trace_end(void* out, int cap, int* n);
#ifdef __cplusplus
}
#endif
#endif
