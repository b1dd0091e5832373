// Internal launchers for the importance kernels (importance.cu), shared with
// the device engine (engine.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace kvp {

constexpr int kMaxTiers = 8;

struct TierParams {
  int bounds[kMaxTiers + 1];  // cumulative group sizes (sorted-rank boundaries)
  int rank_k[kMaxTiers];
  int rank_v[kMaxTiers];
};

TierParams make_tier_params(int n, int n_groups, const double* ratios, const int32_t* key_ranks,
                            const int32_t* value_ranks);
void launch_tiers(int n_tables, int n, const double* scores, long stride, int n_groups, const TierParams& tp,
                  uint8_t* tier_out, uint16_t* rk_out, uint16_t* rv_out, cudaStream_t s);
// scores: n_tables rows of n, row stride score_stride (-1 = n).
void launch_ema(int n_tables, int n, double* scores, int tq, const double* attn, double alpha,
                unsigned* bad_rows, cudaStream_t s, long score_stride = -1);
// |row sum - 1| > 1e-4 or non-finite rows of attn [rows][n] counted into *bad.
void launch_row_check(int rows, int n, const double* attn, unsigned* bad, cudaStream_t s);

}  // namespace kvp
