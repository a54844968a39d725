// Shared device/host helpers for the sm_100a Liger hot-path kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <string>
#include <algorithm>
#include <cmath>
#include <atomic>
#include <mutex>
#include <unordered_map>
#include <type_traits>

#include "../../include/liger_b200.h"

namespace lk {

// ---------------------------------------------------------------- errors ----
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

#define LK_REQUIRE(cond, code, msg)          \
  do {                                       \
    if (!(cond)) return ::lk::fail(code, msg); \
  } while (0)

#define LK_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess)                                                         \
      return ::lk::fail(LK_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// RAII stage timer for lk_profile_* (no-op unless profiling is enabled).
class ProfScope {
 public:
  ProfScope(int stage, cudaStream_t st);
  ~ProfScope();
  ProfScope(const ProfScope&) = delete;
  ProfScope& operator=(const ProfScope&) = delete;

 private:
  int stage_;
  cudaStream_t st_;
  bool active_ = false;
  cudaEvent_t a_{}, b_{};
  int64_t mark_ = 0;
};

// Test-only path knobs (lk_test_select_path, capi.cu); 0 = the product path.
int path_knob(int knob);
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int sm_count() {  // of the current device; cached per device, thread-safe
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel (per size increase).
inline cudaError_t ensure_smem(const void* fn, int bytes) {  // per (kernel, device): attributes are per device
  static std::mutex mu;
  static std::unordered_map<uint64_t, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = reinterpret_cast<uint64_t>(fn) * 64u + (uint64_t)dev;
  std::lock_guard<std::mutex> g(mu);
  int& have = done[key];
  if (have >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller workspace (the library never allocates).
struct Carver {
  char* base;
  size_t cap;
  size_t off = 0;
  Carver(void* p, size_t c) : base(static_cast<char*>(p)), cap(c) {}
  template <typename T>
  T* take(size_t count, size_t align = 256) {
    off = align_up(off, align);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
};

// ------------------------------------------------------ element access ----
template <typename T> struct Elem;
template <> struct Elem<float> {
  static __device__ __forceinline__ float to_f(float v) { return v; }
  static __device__ __forceinline__ float from_f(float v) { return v; }
};
template <> struct Elem<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};
template <> struct Elem<__half> {
  static __device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
  static __device__ __forceinline__ __half from_f(float v) { return __float2half_rn(v); }
};

template <typename T> __device__ __forceinline__ float to_f(T v) { return Elem<T>::to_f(v); }
template <typename T> __device__ __forceinline__ T from_f(float v) { return Elem<T>::from_f(v); }
// round-trip through T (models a cast to the storage dtype)
template <typename T> __device__ __forceinline__ float round_to(float v) { return to_f<T>(from_f<T>(v)); }
// bf16 round-to-nearest-even on the integer pipe (3 ALU ops) instead of an F2F + unpack on the
// 16/clk conversion pipe; exact for all finite values and +-inf (NaNs stay NaN unless their
// payload sits only in the low 16 bits).
template <> __device__ __forceinline__ float round_to<__nv_bfloat16>(float v) {
  uint32_t u = __float_as_uint(v);
  u += 0x7fffu + ((u >> 16) & 1u);
  return __uint_as_float(u & 0xffff0000u);
}

// 16-byte vector of T, unpacked to float.
template <typename T> struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
  float v[N];
  __device__ __forceinline__ void load(const T* p) {
    uint4 raw = *reinterpret_cast<const uint4*>(p);
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = to_f<T>(e[i]);
  }
  __device__ __forceinline__ void load_nc(const T* p) {
    uint4 raw;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w) : "l"(p));
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = to_f<T>(e[i]);
  }
  __device__ __forceinline__ void store(T* p) const {
    uint4 raw;
    if constexpr (sizeof(T) == 2) {  // one F2FP.PACK_AB per pair (a per-element F2F is 4x the work)
      uint32_t* w = reinterpret_cast<uint32_t*>(&raw);
#pragma unroll
      for (int i = 0; i < N / 2; ++i) {
        if constexpr (std::is_same<T, __nv_bfloat16>::value) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&h);
        } else {
          __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&h);
        }
      }
    } else {
      T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
      for (int i = 0; i < N; ++i) e[i] = from_f<T>(v[i]);
    }
    *reinterpret_cast<uint4*>(p) = raw;
  }
};

// --------------------------------------------------------- reductions ----
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
// online-softmax pair combine: (m, s) ⊕ (m2, s2)
__device__ __forceinline__ void ms_combine(float& m, float& s, float m2, float s2) {
  float mn = fmaxf(m, m2);
  if (mn == -INFINITY) { m = mn; s = 0.f; return; }
  s = s * __expf(m - mn) + s2 * __expf(m2 - mn);
  m = mn;
}
__device__ __forceinline__ void warp_ms(float& m, float& s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    ms_combine(m, s, m2, s2);
  }
}

// Block-wide sum; all threads get the result.  scratch: >= 32 floats.
__device__ __forceinline__ float block_sum(float v, float* scratch) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  float r = (lane < nw) ? scratch[lane] : 0.f;
  r = warp_sum(r);
  return r;
}

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace lk

// dtype dispatch helper
#define LK_DISPATCH_FLOAT(dtype, T, ...)                                   \
  switch (dtype) {                                                         \
    case LK_F32: { using T = float; __VA_ARGS__; break; }                  \
    case LK_BF16: { using T = __nv_bfloat16; __VA_ARGS__; break; }         \
    case LK_F16: { using T = __half; __VA_ARGS__; break; }                 \
    default: return ::lk::fail(LK_INVALID_ARGUMENT, "unknown dtype");      \
  }
