// Internal: batched retrieval-plan attention (attend_plan.cu), shared with the
// device LayerCache batch (cache.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kvp_b200.h"

namespace kvp {

struct PlanBatch {
  int heads, kv_heads, head_dim, dtype;
  int batch;       // instances, each with its own plan over the same store structure
  int n_stores;    // stores per instance
  int n_entries;   // plan entries per instance
  int tq;
  int table_size;  // importance-table width (head_avg_table), 0 = none
  long table_stride;
  const kvp_store* stores;          // [host] batch x n_stores
  const kvp_plan_entry* entries;    // batch x n_entries, [dev] when entries_on_device else [host]
  bool entries_on_device;
  const double* queries;            // [dev] batch x tq x H*D
  const uint64_t* query_positions;  // [dev] tq
  double* context;                  // [dev] batch x tq x H*D
  double* head_avg;                 // [dev] batch x tq x n_entries (nullable)
  double* head_avg_table;           // [dev] batch x tq x table_stride (nullable)
};

void run_plan(const PlanBatch& d, cudaStream_t s);

}  // namespace kvp
