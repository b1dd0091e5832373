// Prefill-time compaction of the engine's visual segments (compact.cu).
#pragma once

#include "kvp_b200.h"

namespace kvp {
// Generates every layer's visual K/V prefill (latent-factor model, Philox) and
// factors it in place into the engine's left/right buffers.
void compact_visual(kvp_engine* e);
}  // namespace kvp
