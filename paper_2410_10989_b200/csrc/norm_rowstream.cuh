// RMSNorm warp-per-row streaming kernels (the default path for 16-byte aligned rows).
//
// Each warp owns a row at a time and a private ring of shared-memory stages filled by
// 1D TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx), so the next rows of a
// warp are in flight while the current one is reduced (warp shuffles only, no block
// barrier) and written.  Forward: 12 warps x 2 stages x one row = 24 rows in flight or
// computing per SM.  Backward: 6 warps x 2 stages x (dy row + x row); the dgamma partial
// lives in registers per lane (fixed columns), and the CTA's warps combine their partials
// in a fixed order in shared memory at the end -> one partial row per CTA, then the
// deterministic column sum (rowfuse's _tree_sum role, rowfuse/ops.py:138-152).
#pragma once
#include "common.cuh"

namespace lk {
namespace rs {

constexpr int FWD_WARPS = 12, BWD_WARPS = 6, STAGES = 2;

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(s_u32(b)), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(bar)) : "memory");
}
template <typename T>
__device__ __forceinline__ void ld_vec(const T* p, float (&v)[Vec16<T>::N]) {
  uint4 raw = *reinterpret_cast<const uint4*>(p);
  const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
  for (int i = 0; i < Vec16<T>::N; ++i) v[i] = to_f<T>(e[i]);
}
__host__ __device__ inline uint32_t pad128(uint64_t b) { return (uint32_t)((b + 127) / 128 * 128); }

template <typename T>
__device__ __forceinline__ float fwd_value(float x, float r, float w, bool has_w, float offset, int mode) {
  float xh = x * r;
  if (mode != LK_CAST_GEMMA) xh = round_to<T>(xh);
  return has_w ? xh * (offset + w) : xh;
}

template <typename T, typename R>
__global__ void __launch_bounds__(FWD_WARPS * 32, 1)
rmsnorm_fwd_warp(const T* __restrict__ x, const T* __restrict__ w, T* __restrict__ y, R* __restrict__ rstd,
                 int64_t rows, int64_t cols, float eps, float offset, int mode) {
  constexpr int NV = Vec16<T>::N;
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t rb = (uint32_t)(cols * sizeof(T)), sb = pad128(rb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* wsm = reinterpret_cast<T*>(sm);
  uint8_t* ring = sm + sb + (size_t)warp * STAGES * sb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + sb + (size_t)FWD_WARPS * STAGES * sb) + warp * STAGES;
  const int64_t nvec = cols / NV;
  if (w)
    for (int64_t i = threadIdx.x; i < nvec; i += blockDim.x)
      reinterpret_cast<uint4*>(wsm)[i] = reinterpret_cast<const uint4*>(w)[i];
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t gw = (int64_t)blockIdx.x * FWD_WARPS + warp, GW = (int64_t)gridDim.x * FWD_WARPS;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) {
      const int64_t row = gw + s * GW;
      if (row < rows) { expect_tx(&bars[s], rb); bulk_g2s(ring + s * sb, x + row * cols, rb, &bars[s]); }
    }
  int s = 0;
  uint32_t phase = 0;
  for (int64_t row = gw; row < rows; row += GW) {
    const T* xs = reinterpret_cast<const T*>(ring + s * sb);
    wait(&bars[s], phase);
    float ss = 0.f;
    for (int64_t i = lane; i < nvec; i += 32) {
      float v[NV];
      ld_vec<T>(xs + i * NV, v);
#pragma unroll
      for (int e = 0; e < NV; ++e) ss = fmaf(v[e], v[e], ss);
    }
    ss = warp_sum(ss);
    const float r = rsqrtf(ss / (float)cols + eps);
    if (lane == 0) rstd[row] = from_f<R>(r);
    T* yr = y + row * cols;
    for (int64_t i = lane; i < nvec; i += 32) {
      float v[NV], wv[NV];
      ld_vec<T>(xs + i * NV, v);
      if (w) ld_vec<T>(wsm + i * NV, wv);
      Vec16<T> o;
#pragma unroll
      for (int e = 0; e < NV; ++e) o.v[e] = fwd_value<T>(v[e], r, w ? wv[e] : 0.f, w != nullptr, offset, mode);
      o.store(yr + i * NV);
    }
    __syncwarp();
    if (lane == 0) {
      const int64_t nxt = row + STAGES * GW;
      if (nxt < rows) { expect_tx(&bars[s], rb); bulk_g2s(ring + s * sb, x + nxt * cols, rb, &bars[s]); }
    }
    if (++s == STAGES) { s = 0; phase ^= 1; }
  }
}

// KPL = 16-byte vectors per lane per row (compile time: the dgamma partial lives in registers).
template <typename T, typename R, int KPL>
__global__ void __launch_bounds__(BWD_WARPS * 32, 1)
rmsnorm_bwd_warp(const T* dy, const T* __restrict__ x, const T* __restrict__ w, const R* __restrict__ rstd, T* dx,
                 float* __restrict__ dw_part, int64_t rows, int64_t cols, float offset, int mode) {
  constexpr int NV = Vec16<T>::N;
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t rb = (uint32_t)(cols * sizeof(T)), sb = pad128(rb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* wsm = reinterpret_cast<T*>(sm);
  uint8_t* ring0 = sm + sb;
  uint8_t* ring = ring0 + (size_t)warp * STAGES * 2 * sb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring0 + (size_t)BWD_WARPS * STAGES * 2 * sb) + warp * STAGES;
  const int64_t nvec = cols / NV;
  float acc[KPL][NV];
#pragma unroll
  for (int k = 0; k < KPL; ++k)
#pragma unroll
    for (int e = 0; e < NV; ++e) acc[k][e] = 0.f;
  if (w)
    for (int64_t i = threadIdx.x; i < nvec; i += blockDim.x)
      reinterpret_cast<uint4*>(wsm)[i] = reinterpret_cast<const uint4*>(w)[i];
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t gw = (int64_t)blockIdx.x * BWD_WARPS + warp, GW = (int64_t)gridDim.x * BWD_WARPS;
  auto issue = [&](int s, int64_t row) {
    uint8_t* st = ring + (size_t)s * 2 * sb;
    expect_tx(&bars[s], 2 * rb);
    bulk_g2s(st, dy + row * cols, rb, &bars[s]);
    bulk_g2s(st + sb, x + row * cols, rb, &bars[s]);
  };
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) {
      const int64_t row = gw + s * GW;
      if (row < rows) issue(s, row);
    }
  int s = 0;
  uint32_t phase = 0;
  for (int64_t row = gw; row < rows; row += GW) {
    const T* gs = reinterpret_cast<const T*>(ring + (size_t)s * 2 * sb);
    const T* xs = reinterpret_cast<const T*>(ring + (size_t)s * 2 * sb + sb);
    const float r = to_f<R>(rstd[row]);
    wait(&bars[s], phase);
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const int64_t i = lane + 32 * k;
      if (i < nvec) {
        float g[NV], xv[NV], wv[NV];
        ld_vec<T>(gs + i * NV, g);
        ld_vec<T>(xs + i * NV, xv);
        if (w) ld_vec<T>(wsm + i * NV, wv);
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          float mm = w ? g[e] * (offset + wv[e]) : g[e];
          if (mode == LK_CAST_LLAMA) mm = round_to<T>(mm);
          dot = fmaf(mm, xv[e], dot);
          float xh = xv[e] * r;
          if (mode == LK_CAST_LLAMA) xh = round_to<T>(xh);
          acc[k][e] = fmaf(g[e], xh, acc[k][e]);
        }
      }
    }
    dot = warp_sum(dot);
    const float c = r * r * r * dot / (float)cols;
    T* dxr = dx + row * cols;
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const int64_t i = lane + 32 * k;
      if (i < nvec) {
        float g[NV], xv[NV], wv[NV];
        ld_vec<T>(gs + i * NV, g);
        ld_vec<T>(xs + i * NV, xv);
        if (w) ld_vec<T>(wsm + i * NV, wv);
        Vec16<T> o;
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          float mm = w ? g[e] * (offset + wv[e]) : g[e];
          if (mode == LK_CAST_LLAMA) mm = round_to<T>(mm);
          o.v[e] = r * mm - c * xv[e];
        }
        o.store(dxr + i * NV);
      }
    }
    __syncwarp();
    if (lane == 0) {
      const int64_t nxt = row + STAGES * GW;
      if (nxt < rows) issue(s, nxt);
    }
    if (++s == STAGES) { s = 0; phase ^= 1; }
  }
  if (!dw_part) return;
  // combine the warps' partials in a fixed order: stage each warp's row in smem (ring reuse)
  __syncthreads();
  float* red = reinterpret_cast<float*>(ring0);
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    const int64_t i = lane + 32 * k;
    if (i < nvec)
#pragma unroll
      for (int e = 0; e < NV; e += 4)
        *reinterpret_cast<float4*>(red + (size_t)warp * cols + i * NV + e) =
            make_float4(acc[k][e], acc[k][e + 1], acc[k][e + 2], acc[k][e + 3]);
  }
  __syncthreads();
  float* p = dw_part + (int64_t)blockIdx.x * cols;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int ww = 0; ww < BWD_WARPS; ++ww) t += red[(size_t)ww * cols + c];
    p[c] = t;
  }
}

inline size_t fwd_smem(int64_t cols, int esz) {
  const size_t sb = pad128((uint64_t)cols * esz);
  return sb + (size_t)FWD_WARPS * STAGES * sb + (size_t)FWD_WARPS * STAGES * 8;
}
inline size_t bwd_smem(int64_t cols, int esz) {
  const size_t sb = pad128((uint64_t)cols * esz);
  size_t ring = (size_t)BWD_WARPS * STAGES * 2 * sb;
  const size_t red = (size_t)BWD_WARPS * cols * 4;  // end-of-kernel reuse of the rings
  if (ring < red) ring = red;
  return sb + ring + (size_t)BWD_WARPS * STAGES * 8;
}

}  // namespace rs
}  // namespace lk
