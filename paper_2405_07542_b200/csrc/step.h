// Device argument block of one verify step (all pointers are device memory).
#pragma once
#include "common.h"

namespace sdb {

struct StepArgs {
    int B, cap, layout, stop_on_eos, acc_stride;
    // inputs
    const int32_t* last;     // [B]
    const int32_t* counts;   // [B] draft counts k_s
    const int32_t* drafts;   // concatenated drafts
    const int32_t* budget;   // [B] max_new_tokens - generated
    const int32_t* active;   // [B]
    // cache descriptors (mutated by k_accept)
    int32_t* committed;      // [B]
    int32_t* logical;        // [B]
    uint8_t* pad;            // [B*cap] or null (unpad)
    // pack outputs / scratch
    int32_t* tokens;         // [T_max]
    Plan* plans;             // [T_max]
    int32_t* first_row;      // [B]
    int32_t* draft_off;      // [B]
    int32_t* scalars;        // [0]=T [1]=k_max [2]=grid base [3]=tau_max
    // forward output
    const int32_t* argmax;   // [T_max]
    // accept outputs
    int32_t* tau;            // [B]
    int32_t* accepted;       // [B][acc_stride]
    int32_t* clipped;        // [B]
};

void launch_pack(const StepArgs& a, cudaStream_t st);
void launch_accept(const StepArgs& a, cudaStream_t st);
void launch_pad_fill(const StepArgs& a, const Cache& c, cudaStream_t st);

}  // namespace sdb
