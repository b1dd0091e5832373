// Prefill compaction on the GPU (randomized truncated SVD, linalg.cpp:68-105).
#include "common.cuh"
#include "compact.cuh"

namespace kvp {
void compact_visual(kvp_engine*) { fail(KVP_ERR_PARAMETER, "compaction: not available yet (use factor_init = 1)"); }
}  // namespace kvp
