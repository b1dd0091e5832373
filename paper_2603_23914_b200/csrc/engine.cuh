// Internal: the engine object is defined in engine.cu; compaction (compact.cu)
// receives it opaquely through this header.
#pragma once

#include "kvp_b200.h"
