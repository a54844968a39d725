// RMSNorm fast paths for 16-byte aligned rows (the common case).
//
// Forward: one warp per row, the whole row held in registers as packed 16-bit pairs
// (H = 4096 bf16 -> 16 x 16-byte vectors = 64 registers per lane), all loads of a
// row issued before the shuffle reduction, no block barrier; ~20 warps per SM keep
// ~160 KB of rows in flight.
// Backward: each thread owns VPT 16-byte column vectors; a CTA processes 8 / VPT rows per
// iteration (all their (dy, x) loads in flight per thread, one block reduction per group),
// the dgamma partial stays in registers (VPT x 8 floats) and is written once per CTA;
// the deterministic fixed-order column sum follows (rowfuse's _tree_sum role,
// rowfuse/ops.py:138-152).
#pragma once
#include "common.cuh"

namespace lk {
namespace rs {

constexpr int FWD_THREADS = 128;  // 4 warps = 4 rows per CTA
constexpr int BWD_THREADS = 512;

template <typename T>
__device__ __forceinline__ float fwd_value(float x, float r, float w, bool has_w, float offset, int mode) {
  float xh = x * r;
  if (mode != LK_CAST_GEMMA) xh = round_to<T>(xh);
  return has_w ? xh * (offset + w) : xh;
}
template <typename T>
__device__ __forceinline__ void unpack(const uint4& raw, float (&v)[Vec16<T>::N]) {
  const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
  for (int i = 0; i < Vec16<T>::N; ++i) v[i] = to_f<T>(e[i]);
}

// VPL = 16-byte vectors per lane (compile time; row = VPL * 32 vectors).
template <typename T, typename R, int VPL>
__global__ void __launch_bounds__(FWD_THREADS)
rmsnorm_fwd_warp(const T* __restrict__ x, const T* __restrict__ w, T* __restrict__ y, R* __restrict__ rstd,
                 int64_t rows, int64_t cols, float eps, float offset, int mode) {
  constexpr int NV = Vec16<T>::N;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = cols / NV;
  const int64_t row = (int64_t)blockIdx.x * (FWD_THREADS / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  uint4 raw[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int64_t i = lane + 32 * k;
    if (i < nvec) {
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(raw[k].x), "=r"(raw[k].y), "=r"(raw[k].z), "=r"(raw[k].w) : "l"(xr + i));
    } else {
      raw[k] = make_uint4(0, 0, 0, 0);
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    float v[NV];
    unpack<T>(raw[k], v);
#pragma unroll
    for (int e = 0; e < NV; ++e) ss = fmaf(v[e], v[e], ss);
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / (float)cols + eps);
  if (lane == 0) rstd[row] = from_f<R>(r);
  T* yr = y + row * cols;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int64_t i = lane + 32 * k;
    if (i < nvec) {
      float v[NV], wv[NV];
      unpack<T>(raw[k], v);
      if (w) unpack<T>(reinterpret_cast<const uint4*>(w)[i], wv);
      Vec16<T> o;
#pragma unroll
      for (int e = 0; e < NV; ++e) o.v[e] = fwd_value<T>(v[e], r, w ? wv[e] : 0.f, w != nullptr, offset, mode);
      o.store(yr + i * NV);
    }
  }
}

template <typename T, typename R, int VPT, int BWD_ROWS>
__global__ void __launch_bounds__(BWD_THREADS, 1)
rmsnorm_bwd_rows(const T* dy, const T* __restrict__ x, const T* __restrict__ w, const R* __restrict__ rstd, T* dx,
                 float* __restrict__ dw_part, int64_t rows, int64_t cols, float offset, int mode) {
  constexpr int NV = Vec16<T>::N;
  __shared__ float red[BWD_ROWS][BWD_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nvec = cols / NV;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float acc[VPT][NV];
#pragma unroll
  for (int k = 0; k < VPT; ++k)
#pragma unroll
    for (int e = 0; e < NV; ++e) acc[k][e] = 0.f;
  // gamma is re-read per use (L1-resident, 8 KB at H=4096) to keep registers for the row data
  auto wvec = [&](int64_t i, float (&wv)[NV]) {
    if (w && i < nvec) {
      unpack<T>(__ldg(reinterpret_cast<const uint4*>(w) + i), wv);
#pragma unroll
      for (int e = 0; e < NV; ++e) wv[e] += offset;
    } else {
#pragma unroll
      for (int e = 0; e < NV; ++e) wv[e] = 0.f;  // idle columns: 0 * garbage would be NaN in the row dot
    }
  };
  for (int64_t rb = r0; rb < r1; rb += BWD_ROWS) {
    uint4 gr[BWD_ROWS][VPT], xr[BWD_ROWS][VPT];
    float rr[BWD_ROWS];
#pragma unroll
    for (int j = 0; j < BWD_ROWS; ++j) {
      const int64_t row = rb + j;
      rr[j] = row < r1 ? to_f<R>(rstd[row]) : 0.f;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int64_t i = tid + (int64_t)k * BWD_THREADS;
        if (row < r1 && i < nvec) {
          gr[j][k] = reinterpret_cast<const uint4*>(dy + row * cols)[i];
          xr[j][k] = reinterpret_cast<const uint4*>(x + row * cols)[i];
        } else {
          gr[j][k] = make_uint4(0, 0, 0, 0);
          xr[j][k] = make_uint4(0, 0, 0, 0);
        }
      }
    }
    float dot[BWD_ROWS];
#pragma unroll
    for (int j = 0; j < BWD_ROWS; ++j) {
      dot[j] = 0.f;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        float g[NV], xv[NV], wv[NV];
        unpack<T>(gr[j][k], g);
        unpack<T>(xr[j][k], xv);
        wvec(tid + (int64_t)k * BWD_THREADS, wv);
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          float mm = w ? g[e] * wv[e] : g[e];
          if (mode == LK_CAST_LLAMA) mm = round_to<T>(mm);
          dot[j] = fmaf(mm, xv[e], dot[j]);
          float xh = xv[e] * rr[j];
          if (mode == LK_CAST_LLAMA) xh = round_to<T>(xh);
          acc[k][e] = fmaf(g[e], xh, acc[k][e]);
        }
      }
      dot[j] = warp_sum(dot[j]);
    }
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < BWD_ROWS; ++j) red[j][warp] = dot[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < BWD_ROWS; ++j) {
      float t = lane < BWD_THREADS / 32 ? red[j][lane] : 0.f;
      dot[j] = warp_sum(t);
    }
    __syncthreads();  // red reused next iteration
#pragma unroll
    for (int j = 0; j < BWD_ROWS; ++j) {
      const int64_t row = rb + j;
      if (row >= r1) continue;
      const float r = rr[j];
      const float c = r * r * r * dot[j] / (float)cols;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int64_t i = tid + (int64_t)k * BWD_THREADS;
        if (i < nvec) {
          float g[NV], xv[NV], wv[NV];
          unpack<T>(gr[j][k], g);
          unpack<T>(xr[j][k], xv);
          wvec(i, wv);
          Vec16<T> o;
#pragma unroll
          for (int e = 0; e < NV; ++e) {
            float mm = w ? g[e] * wv[e] : g[e];
            if (mode == LK_CAST_LLAMA) mm = round_to<T>(mm);
            o.v[e] = r * mm - c * xv[e];
          }
          o.store(dx + row * cols + i * NV);
        }
      }
    }
  }
  if (dw_part) {
    float* p = dw_part + (int64_t)blockIdx.x * cols;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int64_t i = tid + (int64_t)k * BWD_THREADS;
      if (i < nvec)
#pragma unroll
        for (int e = 0; e < NV; e += 4)
          *reinterpret_cast<float4*>(p + i * NV + e) = make_float4(acc[k][e], acc[k][e + 1], acc[k][e + 2], acc[k][e + 3]);
    }
  }
}

}  // namespace rs
}  // namespace lk
