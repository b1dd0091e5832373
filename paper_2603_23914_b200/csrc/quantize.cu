// 4-bit groupwise quantisation round trip on the device: quantize_4bit + dequantize
// (quantize.hpp:14-49, quantize.cpp:10-54) behind the Python surface's
// quantize_roundtrip (bindings/module.cpp:223-230).
//
// Per column j and row group g (group_size rows): mn / mx over the group, scale =
// (mx - mn) / 15 (0 for a constant group), code = clamp(lround((v - mn) / scale), 0, 15),
// value = mn + scale * code.  One warp per (column, group); fp64 with the reference's
// operation order (no contraction: __dmul_rn / __dadd_rn), so the result is bit-identical.
#include <cuda_runtime.h>

#include "common.cuh"

namespace kvp {
namespace {

__global__ void quantize_roundtrip_kernel(const double* __restrict__ a, long rows, long cols, long group,
                                          double* __restrict__ out) {
  const long groups = (rows + group - 1) / group;
  const long wid = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= cols * groups) return;
  const long j = wid / groups, g = wid % groups;
  const long lo = g * group, hi = min(lo + group, rows);
  // std::min / std::max sweep (quantize.cpp:23-29) keeps the earliest of equal values (-0 vs +0):
  // reduce (value, row) pairs, ties to the lower row
  double mn = a[lo * cols + j], mx = mn;
  long imn = lo, imx = lo;
  for (long i = lo + lane; i < hi; i += 32) {
    const double v = a[i * cols + j];
    if (v < mn || (v == mn && i < imn)) {
      mn = v;
      imn = i;
    }
    if (mx < v || (v == mx && i < imx)) {
      mx = v;
      imx = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double omn = __shfl_xor_sync(0xffffffffu, mn, o), omx = __shfl_xor_sync(0xffffffffu, mx, o);
    const long oimn = __shfl_xor_sync(0xffffffffu, imn, o), oimx = __shfl_xor_sync(0xffffffffu, imx, o);
    if (omn < mn || (omn == mn && oimn < imn)) {
      mn = omn;
      imn = oimn;
    }
    if (mx < omx || (omx == mx && oimx < imx)) {
      mx = omx;
      imx = oimx;
    }
  }
  const double scale = __ddiv_rn(__dsub_rn(mx, mn), 15.0);
  for (long i = lo + lane; i < hi; i += 32) {
    long code = 0;
    if (scale > 0.0) {
      const long c = llround(__ddiv_rn(__dsub_rn(a[i * cols + j], mn), scale));
      code = c < 0 ? 0 : (c > 15 ? 15 : c);
    }
    out[i * cols + j] = __dadd_rn(mn, __dmul_rn(scale, static_cast<double>(code)));
  }
}

}  // namespace
}  // namespace kvp

// quantize_roundtrip (module.cpp:223-230): a, out [dev] row-major f64 rows x cols.
extern "C" int kvp_quantize_roundtrip(const double* a, int64_t rows, int64_t cols, int64_t group_size, double* out,
                                      void* stream) {
  return kvp::guarded([&] {
    using namespace kvp;
    require(group_size >= 1, KVP_ERR_PARAMETER, "quantize_4bit: group_size must be >= 1");
    require(rows >= 0 && cols >= 0, KVP_ERR_SHAPE, "quantize_4bit: negative shape");
    require(a != nullptr && out != nullptr, KVP_ERR_PARAMETER, "quantize_4bit: null buffer");
    if (rows == 0 || cols == 0) return;
    const long warps = cols * ((rows + group_size - 1) / group_size);
    quantize_roundtrip_kernel<<<cdiv(warps * 32, 256), 256, 0, as_stream(stream)>>>(a, rows, cols, group_size, out);
    KVP_LAUNCHED();
  });
}
