// Shared helpers for the kvrerank_b200 CUDA library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>
#include <atomic>

#include "../../include/kvrerank_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "kvrerank_b200 is written for sm_100a only"
#endif

namespace krr {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
std::atomic<uint64_t>& launch_counter();

// Checks the launch that was just queued; counts it.
int check_launch(const char* what);

// Per-device, thread-safe launch setup (a process may drive several GPUs from
// several threads): SM count of the current device; the dynamic-smem opt-in
// (and carveout, when >= 0) of a kernel applied once per (device, kernel);
// an int computed once per (device, key) -- e.g. co-resident cluster counts.
int current_device();
int device_sm_count();
int ensure_func_smem(const void* func, int smem_bytes, int carveout = -1);
int cached_per_device(const void* key, int (*compute)(const void* ctx), const void* ctx);

#define KRR_REQUIRE(cond, code, msg)            \
  do {                                          \
    if (!(cond)) return ::krr::fail(code, msg); \
  } while (0)

// ---------------------------------------------------------------- dtypes
template <typename T> struct Act;
template <> struct Act<float> {
  static constexpr int code = KRR_F32;
  __device__ static inline float from(float v) { return v; }
  __device__ static inline float to(float v) { return v; }
};
template <> struct Act<__half> {
  static constexpr int code = KRR_F16;
  __device__ static inline __half from(float v) { return __float2half_rn(v); }
  __device__ static inline float to(__half v) { return __half2float(v); }
};
template <> struct Act<__nv_bfloat16> {
  static constexpr int code = KRR_BF16;
  __device__ static inline __nv_bfloat16 from(float v) { return __float2bfloat16_rn(v); }
  __device__ static inline float to(__nv_bfloat16 v) { return __bfloat162float(v); }
};

inline size_t dtype_size(int dt) { return dt == KRR_F32 ? 4 : 2; }

// tanh GELU with the reference constants (model.py:34-35, 444-446)
__device__ __forceinline__ float gelu_tanh(float x) {
  const float a = 0.7978845608028654f;  // sqrt(2/pi) as float32
  const float b = 0.044715f;
  float inner = a * (x + b * x * x * x);
  return 0.5f * x * (1.0f + tanhf(inner));
}

// SiLU for the SwiGLU variant: x * sigmoid(x)
__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Profiling hooks used by krr_forward (kernel classes: 0 gemm, 1 attention, 2 misc).
struct ProfScope {
  cudaStream_t s;
  int cls;
  double flops;
  bool on;
  cudaEvent_t e0, e1;
  ProfScope(cudaStream_t s_, int cls_, double flops_ = 0.0);
  ~ProfScope();
};

}  // namespace krr
