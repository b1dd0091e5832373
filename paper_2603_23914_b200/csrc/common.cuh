// Shared plumbing for the B200 kernels: status/error state, launch
// accounting, dtype helpers.  Everything here is internal to libkvp_b200.so.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "kvp_b200.h"

namespace kvp {

// Typed failures thrown inside the library and converted to kvp_status at the
// C-ABI edge (capi.cu).  They mirror kvpack::parameter_error / shape_error /
// data_error / io_error (errors.hpp:11-36).
struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Failure(code, m); }
inline void require(bool ok, int code, const char* m) {
  if (!ok) fail(code, m);
}

void set_last_error(const std::string& m);
void note_launch(uint64_t n = 1);

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(KVP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define KVP_CUDA(x) ::kvp::cuda_check((x), #x)
// Launch bookkeeping: count the launch and surface configuration errors.
#define KVP_LAUNCHED()                                    \
  do {                                                    \
    ::kvp::note_launch();                                 \
    ::kvp::cuda_check(cudaGetLastError(), "kernel launch"); \
  } while (0)

// C-ABI wrapper: run `f`, convert typed failures to status codes.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return KVP_OK;
  } catch (const Failure& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return KVP_ERR_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return KVP_ERR_CUDA;
  }
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// ---- dtype helpers --------------------------------------------------------
__device__ __forceinline__ double to_d(float x) { return static_cast<double>(x); }
__device__ __forceinline__ double to_d(double x) { return x; }
__device__ __forceinline__ double to_d(__nv_bfloat16 x) { return static_cast<double>(__bfloat162float(x)); }
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(double x) { return static_cast<float>(x); }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }

inline size_t dtype_size(int dt) { return dt == KVP_F64 ? 8 : dt == KVP_F32 ? 4 : 2; }

// Stream-ordered scratch allocation released at scope exit.
struct Scratch {
  void* p = nullptr;
  cudaStream_t s;
  Scratch(size_t bytes, cudaStream_t st) : s(st) {
    if (bytes) KVP_CUDA(cudaMallocAsync(&p, bytes, s));
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
};

inline unsigned cdiv(long a, long b) { return static_cast<unsigned>((a + b - 1) / b); }

}  // namespace kvp
