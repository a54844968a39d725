// RMSNorm forward / backward.
//
// Forward (rowfuse/ops.py:190-214; Liger casting modes LK/ops/rms_norm.py:45-112):
//   y = x * rstd * (offset + w), rstd = 1/sqrt(mean(x^2) + eps), one rstd per row cached.
// Backward (rowfuse/ops.py:217-241; LK/ops/rms_norm.py:115-210):
//   dx = rstd * (m - (rstd^2 / n) * (m . x) * x),  m = dy * (offset + w)
//   dw = sum_rows dy * xhat  -- two-stage: one fp32 partial row per CTA, then a
//   fixed-order column sum.  The combine order depends only on the row count and
//   the grid, so the result is bitwise reproducible (the property rowfuse gets from
//   _tree_sum, ops.py:138-152).
//
// One CTA per row in the forward (the row lives in registers between the
// reduction and the write: one read, one write).  The backward is persistent:
// grid = a multiple of the SM count, contiguous row ranges per CTA.
#include "common.cuh"

namespace lk {

template <typename T, bool VEC, int KV>
struct RowIO {
  static constexpr int NV = VEC ? Vec16<T>::N : 1;
  // column of element e of vector slot k for thread tid
  static __device__ __forceinline__ int64_t col(int k, int e, int tid, int bs) {
    return ((int64_t)k * bs + tid) * NV + e;
  }
  static __device__ __forceinline__ void load(const T* p, int64_t cols, float (&v)[KV][NV], int tid, int bs) {
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      int64_t c0 = col(k, 0, tid, bs);
      if (VEC) {
        if (c0 < cols) {
          Vec16<T> t;
          t.load(p + c0);
#pragma unroll
          for (int e = 0; e < NV; ++e) v[k][e] = t.v[e];
        } else {
#pragma unroll
          for (int e = 0; e < NV; ++e) v[k][e] = 0.f;
        }
      } else {
        v[k][0] = c0 < cols ? to_f<T>(p[c0]) : 0.f;
      }
    }
  }
  static __device__ __forceinline__ void store(T* p, int64_t cols, const float (&v)[KV][NV], int tid, int bs) {
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      int64_t c0 = col(k, 0, tid, bs);
      if (c0 >= cols) continue;
      if (VEC) {
        Vec16<T> t;
#pragma unroll
        for (int e = 0; e < NV; ++e) t.v[e] = v[k][e];
        t.store(p + c0);
      } else {
        p[c0] = from_f<T>(v[k][0]);
      }
    }
  }
};

template <typename T, typename R, bool VEC, int KV>
__global__ void rmsnorm_fwd_kernel(const T* __restrict__ x, const T* __restrict__ w, T* __restrict__ y,
                                   R* __restrict__ rstd, int64_t rows, int64_t cols, float eps,
                                   float offset, int mode) {
  using IO = RowIO<T, VEC, KV>;
  constexpr int NV = IO::NV;
  __shared__ float scratch[32];
  const int tid = threadIdx.x, bs = blockDim.x;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    float v[KV][NV];
    IO::load(x + row * cols, cols, v, tid, bs);
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int e = 0; e < NV; ++e) ss += v[k][e] * v[k][e];
    ss = block_sum(ss, scratch);
    const float r = rsqrtf(ss / (float)cols + eps);
    if (tid == 0) rstd[row] = from_f<R>(r);
    float wv[KV][NV];
    if (w) IO::load(w, cols, wv, tid, bs);
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        float xh = v[k][e] * r;
        if (mode != LK_CAST_GEMMA) xh = round_to<T>(xh);  // llama: cast xhat before *w
        v[k][e] = w ? xh * (offset + wv[k][e]) : xh;
      }
    IO::store(y + row * cols, cols, v, tid, bs);
  }
}

template <typename T, typename R, bool VEC, int KV>
__global__ void rmsnorm_bwd_kernel(const T* dy, const T* __restrict__ x,
                                   const T* __restrict__ w, const R* __restrict__ rstd, T* dx,
                                   float* __restrict__ dw_part, int64_t rows, int64_t cols,
                                   float offset, int mode) {
  using IO = RowIO<T, VEC, KV>;
  constexpr int NV = IO::NV;
  __shared__ float scratch[32];
  const int tid = threadIdx.x, bs = blockDim.x;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float wv[KV][NV];
  float acc[KV][NV];
#pragma unroll
  for (int k = 0; k < KV; ++k)
#pragma unroll
    for (int e = 0; e < NV; ++e) acc[k][e] = 0.f;
  if (w) {
    IO::load(w, cols, wv, tid, bs);
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int e = 0; e < NV; ++e) wv[k][e] += offset;
  }
  for (int64_t row = r0; row < r1; ++row) {
    float g[KV][NV], xv[KV][NV];
    IO::load(dy + row * cols, cols, g, tid, bs);
    IO::load(x + row * cols, cols, xv, tid, bs);
    const float r = to_f<R>(rstd[row]);
    float dot = 0.f;
    float m[KV][NV];
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        float mm = w ? g[k][e] * wv[k][e] : g[k][e];
        if (mode == LK_CAST_LLAMA) mm = round_to<T>(mm);  // (dY * W) in x dtype, then fp32
        m[k][e] = mm;
        dot += mm * xv[k][e];
      }
    dot = block_sum(dot, scratch);
    const float c = r * r * r * dot / (float)cols;
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        float xh = xv[k][e] * r;
        if (mode == LK_CAST_LLAMA) xh = round_to<T>(xh);
        acc[k][e] += g[k][e] * xh;
        m[k][e] = r * m[k][e] - c * xv[k][e];
      }
    IO::store(dx + row * cols, cols, m, tid, bs);
  }
  if (dw_part) {
    float* p = dw_part + (int64_t)blockIdx.x * cols;
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        int64_t cidx = IO::col(k, e, tid, bs);
        if (cidx < cols) p[cidx] = acc[k][e];
      }
  }
}

// dw[c] = sum_g part[g, c], fixed order over g (deterministic second stage).
template <typename T>
__global__ void colsum_partials_kernel(const float* __restrict__ part, int64_t g, int64_t cols,
                                       T* __restrict__ out) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int64_t i = 0; i < g; ++i) s += part[i * cols + c];
  out[c] = from_f<T>(s);
}

struct NormCfg {
  bool vec;
  int kv;
  int block;
};

template <typename T>
static NormCfg pick_cfg(int64_t cols, const void* p0, const void* p1, const void* p2) {
  constexpr int NV = Vec16<T>::N;
  bool vec = (cols % NV == 0);
  for (const void* p : {p0, p1, p2})
    if (p && (reinterpret_cast<uintptr_t>(p) & 15)) vec = false;
  int64_t units = vec ? cols / NV : cols;
  int kv = 1;
  while (kv < 8 && (units + kv - 1) / kv > 256) kv *= 2;
  int64_t block = (units + kv - 1) / kv;
  block = std::min<int64_t>(1024, std::max<int64_t>(32, (block + 31) / 32 * 32));
  return {vec, kv, (int)block};
}

#define LK_KV_DISPATCH(kv, KV, ...)                  \
  switch (kv) {                                      \
    case 1: { constexpr int KV = 1; __VA_ARGS__; break; } \
    case 2: { constexpr int KV = 2; __VA_ARGS__; break; } \
    case 4: { constexpr int KV = 4; __VA_ARGS__; break; } \
    default: { constexpr int KV = 8; __VA_ARGS__; break; } \
  }

static int64_t max_cols_for(NormCfg c, int nv) { return (int64_t)c.block * c.kv * (c.vec ? nv : 1); }

}  // namespace lk

using namespace lk;

extern "C" int lk_rmsnorm_fwd(const void* x, const void* weight, void* y, void* rstd, int64_t rows,
                              int64_t cols, float eps, float offset, int casting_mode, int dtype,
                              void* stream) {
  LK_REQUIRE(rows >= 0 && cols >= 1, LK_SIZE_MISMATCH, "rows >= 0 and cols >= 1 required");
  if (rows == 0) return LK_OK;
  LK_REQUIRE(x && y && rstd, LK_INVALID_ARGUMENT, "null pointer");
  LK_REQUIRE(casting_mode >= 0 && casting_mode <= 2, LK_INVALID_ARGUMENT, "bad casting mode");
  cudaStream_t st = as_stream(stream);
  unsigned grid = (unsigned)std::min<int64_t>(rows, 1 << 20);
  LK_DISPATCH_FLOAT(dtype, T, {
    NormCfg c = pick_cfg<T>(cols, x, y, weight);
    LK_REQUIRE(cols <= max_cols_for(c, Vec16<T>::N), LK_SIZE_MISMATCH, "feature dim too large");
    const T* w = static_cast<const T*>(weight);
    if (casting_mode == LK_CAST_NONE) {
      LK_KV_DISPATCH(c.kv, KV, {
        if (c.vec) rmsnorm_fwd_kernel<T, T, true, KV><<<grid, c.block, 0, st>>>(static_cast<const T*>(x), w, static_cast<T*>(y), static_cast<T*>(rstd), rows, cols, eps, offset, casting_mode);
        else rmsnorm_fwd_kernel<T, T, false, KV><<<grid, c.block, 0, st>>>(static_cast<const T*>(x), w, static_cast<T*>(y), static_cast<T*>(rstd), rows, cols, eps, offset, casting_mode);
      });
    } else {
      LK_KV_DISPATCH(c.kv, KV, {
        if (c.vec) rmsnorm_fwd_kernel<T, float, true, KV><<<grid, c.block, 0, st>>>(static_cast<const T*>(x), w, static_cast<T*>(y), static_cast<float*>(rstd), rows, cols, eps, offset, casting_mode);
        else rmsnorm_fwd_kernel<T, float, false, KV><<<grid, c.block, 0, st>>>(static_cast<const T*>(x), w, static_cast<T*>(y), static_cast<float*>(rstd), rows, cols, eps, offset, casting_mode);
      });
    }
  });
  return check_launch("rmsnorm_fwd_kernel");
}

static int64_t rms_bwd_grid(int64_t rows) {
  return std::max<int64_t>(1, std::min<int64_t>(rows, 2 * (int64_t)sm_count()));
}

extern "C" size_t lk_rmsnorm_bwd_workspace_bytes(int64_t rows, int64_t cols) {
  return (size_t)rms_bwd_grid(rows) * (size_t)cols * sizeof(float) + 256;
}

extern "C" int lk_rmsnorm_bwd(const void* dy, const void* x, const void* weight, const void* rstd,
                              void* dx, void* dw, int64_t rows, int64_t cols, float offset,
                              int casting_mode, int dtype, void* workspace, size_t workspace_bytes,
                              void* stream) {
  LK_REQUIRE(rows >= 0 && cols >= 1, LK_SIZE_MISMATCH, "rows >= 0 and cols >= 1 required");
  LK_REQUIRE(casting_mode >= 0 && casting_mode <= 2, LK_INVALID_ARGUMENT, "bad casting mode");
  cudaStream_t st = as_stream(stream);
  const int64_t g = rms_bwd_grid(rows);
  float* part = nullptr;
  if (weight && dw) {
    LK_REQUIRE(workspace && workspace_bytes >= (size_t)g * cols * sizeof(float), LK_INVALID_ARGUMENT,
               "workspace too small");
    part = static_cast<float*>(workspace);
  }
  if (rows == 0) {
    if (part) LK_CUDA(cudaMemsetAsync(part, 0, (size_t)g * cols * sizeof(float), st));
  }
  LK_REQUIRE(rows == 0 || (dy && x && rstd && dx), LK_INVALID_ARGUMENT, "null pointer");
  LK_DISPATCH_FLOAT(dtype, T, {
    if (rows > 0) {
      NormCfg c = pick_cfg<T>(cols, dy, x, dx);
      if (weight && (reinterpret_cast<uintptr_t>(weight) & 15)) c.vec = false;
      LK_REQUIRE(cols <= max_cols_for(c, Vec16<T>::N), LK_SIZE_MISMATCH, "feature dim too large");
      const T* w = static_cast<const T*>(weight);
      if (casting_mode == LK_CAST_NONE) {
        LK_KV_DISPATCH(c.kv, KV, {
          if (c.vec) rmsnorm_bwd_kernel<T, T, true, KV><<<(unsigned)g, c.block, 0, st>>>(static_cast<const T*>(dy), static_cast<const T*>(x), w, static_cast<const T*>(rstd), static_cast<T*>(dx), part, rows, cols, offset, casting_mode);
          else rmsnorm_bwd_kernel<T, T, false, KV><<<(unsigned)g, c.block, 0, st>>>(static_cast<const T*>(dy), static_cast<const T*>(x), w, static_cast<const T*>(rstd), static_cast<T*>(dx), part, rows, cols, offset, casting_mode);
        });
      } else {
        LK_KV_DISPATCH(c.kv, KV, {
          if (c.vec) rmsnorm_bwd_kernel<T, float, true, KV><<<(unsigned)g, c.block, 0, st>>>(static_cast<const T*>(dy), static_cast<const T*>(x), w, static_cast<const float*>(rstd), static_cast<T*>(dx), part, rows, cols, offset, casting_mode);
          else rmsnorm_bwd_kernel<T, float, false, KV><<<(unsigned)g, c.block, 0, st>>>(static_cast<const T*>(dy), static_cast<const T*>(x), w, static_cast<const float*>(rstd), static_cast<T*>(dx), part, rows, cols, offset, casting_mode);
        });
      }
      int rc = check_launch("rmsnorm_bwd_kernel");
      if (rc) return rc;
    }
    if (part) {
      colsum_partials_kernel<T><<<(unsigned)((cols + 255) / 256), 256, 0, st>>>(part, g, cols, static_cast<T*>(dw));
    }
  });
  return check_launch("colsum_partials_kernel");
}
