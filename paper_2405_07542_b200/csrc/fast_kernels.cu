// bf16 performance-mode forward (placeholder until the tcgen05 path lands).
#include "handles.h"

namespace sdb {
void forward_fast(const Model&, Cache&, Workspace&, int, bool, cudaStream_t) {
    throw Error(INTERNAL, "bf16 performance path not built yet");
}
}  // namespace sdb
