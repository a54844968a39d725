// RMSNorm persistent TMA-ring kernels (default path for 16-byte aligned rows).
//
// One CTA per SM = NW consumer warps (NW*32 threads own the row's 16-byte column
// vectors: thread t owns vectors t, t + NW*32, ...) + one producer warp.  A ring stage
// holds RB consecutive rows (forward: x; backward: dy and x), filled by ONE 1D bulk
// copy per tensor (rows are contiguous), so up to S*RB rows per SM are in flight while
// the consumers work on an earlier stage.  Per stage the RB per-row reductions are
// done together: warp shuffles, one named barrier over the consumer warps, then every
// warp sums the per-warp partials in fixed warp order (deterministic, no 2nd barrier;
// the partial buffer is double-buffered by stage parity).
//
// Why this shape (profiles/r01_rowops_ncu.md): warp-per-row kernels (registers or a
// per-warp ring) ran 8-12 warps per SM with long per-row dependency chains and were
// latency-bound at ~1.6 TB/s; column ownership gives 16 warps per SM, a tiny
// per-thread dgamma partial (VPT x 8 floats) and full-row loads in flight.
//
// Backward: each thread's dgamma partial stays in registers and is written once per
// CTA (one partial row per CTA); the fixed-order column sum follows (rowfuse's
// _tree_sum role, rowfuse/ops.py:138-152): bitwise deterministic for a given grid.
#pragma once
#include "ring.cuh"

namespace lk {
namespace rr {

constexpr int MAX_NW = 16;        // consumer warps
constexpr int FWD_RB = 4;         // rows per stage (forward)
constexpr int BWD_RB = 2;         // rows per stage (backward; dy + x)

template <typename T>
__device__ __forceinline__ float fwd_value(float x, float r, float w, bool has_w, float offset, int mode) {
  float xh = x * r;
  if (mode != LK_CAST_GEMMA) xh = round_to<T>(xh);  // llama / none: cast xhat to x dtype before *w
  return has_w ? xh * (offset + w) : xh;
}

// Shared-memory carve-up: [gamma | stages | full[S] | empty[S] | red[2][RB][MAX_NW]]
struct Layout {
  uint32_t gbytes, row_bytes, stage_bytes, ring_off, bar_off, red_off, total;
};
__host__ __device__ inline Layout layout(int64_t cols, int esz, int rows_per_stage, int tensors, int stages) {
  Layout L;
  L.row_bytes = (uint32_t)(cols * esz);
  L.gbytes = ring::pad128(L.row_bytes);
  L.stage_bytes = ring::pad128((uint64_t)L.row_bytes * rows_per_stage * tensors);
  L.ring_off = L.gbytes;
  L.bar_off = L.ring_off + L.stage_bytes * stages;
  L.red_off = L.bar_off + 16 * stages;
  L.total = L.red_off + 2 * rows_per_stage * MAX_NW * 4;
  return L;
}

template <typename T, typename R, int VPT>
__global__ void __launch_bounds__((MAX_NW + 1) * 32, 1)
rmsnorm_fwd_ring(const T* __restrict__ x, const T* __restrict__ w, T* __restrict__ y, R* __restrict__ rstd,
                 int64_t rows, int64_t cols, float eps, float offset, int mode, int stages) {
  constexpr int NV = 16 / sizeof(T);
  constexpr int RB = FWD_RB;
  extern __shared__ __align__(128) uint8_t sm[];
  const Layout L = layout(cols, sizeof(T), RB, 1, stages);
  const int nw = blockDim.x / 32 - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.bar_off);
  uint64_t* empty = full + stages;
  float* red = reinterpret_cast<float*>(sm + L.red_off);  // [2][RB][MAX_NW]
  const int64_t nvec = cols / NV;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t nb = (rows + RB - 1) / RB;
  if (w)
    for (int64_t i = threadIdx.x; i < nvec; i += blockDim.x)
      reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(w)[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { ring::mbar_init(&full[s], 1); ring::mbar_init(&empty[s], nw); }
    ring::fence_init();
  }
  __syncthreads();

  if (warp == nw) {  // producer
    if (lane == 0) {
      ring::Cursor cur(stages);
      for (int64_t k = b; k < nb; k += G, cur.next()) {
        const int s = cur.s;
        if (cur.wrapped) ring::wait(&empty[s], cur.phase ^ 1u);
        const int64_t r0 = k * RB, nr = min((int64_t)RB, rows - r0);
        const uint32_t bytes = (uint32_t)(nr * L.row_bytes);
        ring::expect_tx(&full[s], bytes);
        ring::bulk_g2s(sm + L.ring_off + (size_t)s * L.stage_bytes, x + r0 * cols, bytes, &full[s]);
      }
    }
    return;
  }
  using P = ring::Pairs<T>;
  constexpr int NP = P::NP;
  const int tid = threadIdx.x, nt = nw * 32;
  // bf16, offset 0, xhat rounded to bf16 before *w (llama / none): y = bf16(xhat_bf16 * w) is
  // exactly one packed bf16x2 multiply (the fp32 product of two bf16 values is exact).
  constexpr bool BF16 = std::is_same<T, __nv_bfloat16>::value;
  const bool hmul = BF16 && w != nullptr && offset == 0.f && mode != LK_CAST_GEMMA;
  ring::Cursor cur(stages);
  int par = 1;
  for (int64_t k = b; k < nb; k += G, cur.next()) {
    const int s = cur.s;
    par ^= 1;
    const int64_t r0 = k * RB, nr = min((int64_t)RB, rows - r0);
    const uint8_t* st = sm + L.ring_off + (size_t)s * L.stage_bytes;
    ring::wait(&full[s], cur.phase);
    float ss[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      float2 s2 = make_float2(0.f, 0.f);
      if (j < nr) {
#pragma unroll
        for (int p = 0; p < VPT; ++p) {
          const int64_t v = tid + (int64_t)p * nt;
          if (v < nvec) {
            float2 f[NP];
            P::unpack(ring::lds128(st + j * L.row_bytes + v * 16), f);
#pragma unroll
            for (int e = 0; e < NP; ++e) s2 = __ffma2_rn(f[e], f[e], s2);
          }
        }
      }
      ss[j] = warp_sum(s2.x + s2.y);
    }
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < RB; ++j) red[(par * RB + j) * MAX_NW + warp] = ss[j];
    ring::consumers_sync(1, nt);
    float2 r2[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {  // fixed shuffle tree over the warp partials: deterministic
      const float t = warp_sum(lane < nw ? red[(par * RB + j) * MAX_NW + lane] : 0.f);
      const float r = rsqrtf(t / (float)cols + eps);
      r2[j] = make_float2(r, r);
      if (tid == 0 && j < nr) rstd[r0 + j] = from_f<R>(r);
    }
#pragma unroll
    for (int p = 0; p < VPT; ++p) {
      const int64_t v = tid + (int64_t)p * nt;
      if (v < nvec) {
        uint4 wraw = make_uint4(0, 0, 0, 0);
        float2 wv[NP];
        if (w) {
          wraw = ring::lds128(sm + v * 16);
          P::unpack(wraw, wv);
#pragma unroll
          for (int e = 0; e < NP; ++e) wv[e] = __fadd2_rn(wv[e], make_float2(offset, offset));
        }
#pragma unroll
        for (int j = 0; j < RB; ++j) {
          if (j < nr) {
            float2 f[NP];
            P::unpack(ring::lds128(st + j * L.row_bytes + v * 16), f);
#pragma unroll
            for (int e = 0; e < NP; ++e) f[e] = __fmul2_rn(f[e], r2[j]);
            uint4 out;
            if (hmul) {
              uint4 xb = P::pack(f);  // xhat rounded to bf16
              const uint32_t* xa = reinterpret_cast<const uint32_t*>(&xb);
              const uint32_t* wa = reinterpret_cast<const uint32_t*>(&wraw);
              uint32_t o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 h = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&xa[e]),
                                           *reinterpret_cast<const __nv_bfloat162*>(&wa[e]));
                o[e] = *reinterpret_cast<uint32_t*>(&h);
              }
              out = make_uint4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
              for (int e = 0; e < NP; ++e) {
                if (mode != LK_CAST_GEMMA) f[e] = ring::round2<T>(f[e]);  // llama / none: xhat in x dtype
                if (w) f[e] = __fmul2_rn(f[e], wv[e]);
              }
              out = P::pack(f);
            }
            ring::stg128(y + (r0 + j) * cols + v * NV, out);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) ring::arrive(&empty[s]);
  }
}

template <typename T, typename R, int VPT>
__global__ void __launch_bounds__((MAX_NW + 1) * 32, 1)
rmsnorm_bwd_ring(const T* dy, const T* __restrict__ x, const T* __restrict__ w, const R* __restrict__ rstd, T* dx,
                 float* __restrict__ dw_part, int64_t rows, int64_t cols, float offset, int mode, int stages) {
  constexpr int NV = 16 / sizeof(T);
  constexpr int RB = BWD_RB;
  extern __shared__ __align__(128) uint8_t sm[];
  const Layout L = layout(cols, sizeof(T), RB, 2, stages);
  const int nw = blockDim.x / 32 - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.bar_off);
  uint64_t* empty = full + stages;
  float* red = reinterpret_cast<float*>(sm + L.red_off);
  const int64_t nvec = cols / NV;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t nb = (rows + RB - 1) / RB;
  const uint32_t xoff = RB * L.row_bytes;  // x rows follow the dy rows inside a stage
  if (w)
    for (int64_t i = threadIdx.x; i < nvec; i += blockDim.x)
      reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(w)[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { ring::mbar_init(&full[s], 1); ring::mbar_init(&empty[s], nw); }
    ring::fence_init();
  }
  __syncthreads();

  if (warp == nw) {  // producer
    if (lane == 0) {
      ring::Cursor cur(stages);
      for (int64_t k = b; k < nb; k += G, cur.next()) {
        const int s = cur.s;
        if (cur.wrapped) ring::wait(&empty[s], cur.phase ^ 1u);
        const int64_t r0 = k * RB, nr = min((int64_t)RB, rows - r0);
        const uint32_t bytes = (uint32_t)(nr * L.row_bytes);
        uint8_t* st = sm + L.ring_off + (size_t)s * L.stage_bytes;
        ring::expect_tx(&full[s], 2 * bytes);
        ring::bulk_g2s(st, dy + r0 * cols, bytes, &full[s]);
        ring::bulk_g2s(st + xoff, x + r0 * cols, bytes, &full[s]);
      }
    }
    return;
  }
  using P = ring::Pairs<T>;
  constexpr int NP = P::NP;
  const int tid = threadIdx.x, nt = nw * 32;
  const bool llama = mode == LK_CAST_LLAMA;
  float2 acc[VPT][NP];
#pragma unroll
  for (int p = 0; p < VPT; ++p)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc[p][e] = make_float2(0.f, 0.f);
  // m = dy * (offset + w), rounded to x dtype in llama mode (LK/ops/rms_norm.py:150-170)
  auto mvec = [&](const float2 (&g)[NP], const float2 (&wv)[NP], float2 (&m)[NP]) {
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      m[e] = w ? __fmul2_rn(g[e], wv[e]) : g[e];
      if (llama) m[e] = ring::round2<T>(m[e]);
    }
  };
  ring::Cursor cur(stages);
  int par = 1;
  for (int64_t k = b; k < nb; k += G, cur.next()) {
    const int s = cur.s;
    par ^= 1;
    const int64_t r0 = k * RB, nr = min((int64_t)RB, rows - r0);
    const uint8_t* st = sm + L.ring_off + (size_t)s * L.stage_bytes;
    float2 r2[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const float r = j < nr ? to_f<R>(rstd[r0 + j]) : 0.f;
      r2[j] = make_float2(r, r);
    }
    ring::wait(&full[s], cur.phase);
    // pass 1: dot_j = sum m*x, dgamma partial += dy * xhat
    float2 dot2[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) dot2[j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int p = 0; p < VPT; ++p) {
      const int64_t v = tid + (int64_t)p * nt;
      if (v < nvec) {
        float2 wv[NP];
        if (w) {
          P::unpack(ring::lds128(sm + v * 16), wv);
#pragma unroll
          for (int e = 0; e < NP; ++e) wv[e] = __fadd2_rn(wv[e], make_float2(offset, offset));
        }
#pragma unroll
        for (int j = 0; j < RB; ++j) {
          if (j < nr) {
            float2 g[NP], xv[NP], m[NP];
            P::unpack(ring::lds128(st + j * L.row_bytes + v * 16), g);
            P::unpack(ring::lds128(st + xoff + j * L.row_bytes + v * 16), xv);
            mvec(g, wv, m);
#pragma unroll
            for (int e = 0; e < NP; ++e) {
              dot2[j] = __ffma2_rn(m[e], xv[e], dot2[j]);
              float2 xh = __fmul2_rn(xv[e], r2[j]);
              if (llama) xh = ring::round2<T>(xh);
              acc[p][e] = __ffma2_rn(g[e], xh, acc[p][e]);
            }
          }
        }
      }
    }
    float dsum[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) dsum[j] = warp_sum(dot2[j].x + dot2[j].y);
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < RB; ++j) red[(par * RB + j) * MAX_NW + warp] = dsum[j];
    ring::consumers_sync(1, nt);
    float2 nc2[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {  // fixed shuffle tree over the warp partials: deterministic
      const float t = warp_sum(lane < nw ? red[(par * RB + j) * MAX_NW + lane] : 0.f);
      const float c = r2[j].x * r2[j].x * r2[j].x * t / (float)cols;
      nc2[j] = make_float2(-c, -c);
    }
    // pass 2: dx = r*m - c*x
#pragma unroll
    for (int p = 0; p < VPT; ++p) {
      const int64_t v = tid + (int64_t)p * nt;
      if (v < nvec) {
        float2 wv[NP];
        if (w) {
          P::unpack(ring::lds128(sm + v * 16), wv);
#pragma unroll
          for (int e = 0; e < NP; ++e) wv[e] = __fadd2_rn(wv[e], make_float2(offset, offset));
        }
#pragma unroll
        for (int j = 0; j < RB; ++j) {
          if (j < nr) {
            float2 g[NP], xv[NP], m[NP];
            P::unpack(ring::lds128(st + j * L.row_bytes + v * 16), g);
            P::unpack(ring::lds128(st + xoff + j * L.row_bytes + v * 16), xv);
            mvec(g, wv, m);
#pragma unroll
            for (int e = 0; e < NP; ++e) m[e] = __ffma2_rn(m[e], r2[j], __fmul2_rn(xv[e], nc2[j]));
            ring::stg128(dx + (r0 + j) * cols + v * NV, P::pack(m));
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) ring::arrive(&empty[s]);
  }
  if (!dw_part) return;
  float* pr = dw_part + (int64_t)b * cols;
#pragma unroll
  for (int p = 0; p < VPT; ++p) {
    const int64_t v = tid + (int64_t)p * nt;
    if (v < nvec) {
      float4* q = reinterpret_cast<float4*>(pr + v * NV);
#pragma unroll
      for (int e = 0; e < NP; e += 2) q[e / 2] = make_float4(acc[p][e].x, acc[p][e].y, acc[p][e + 1].x, acc[p][e + 1].y);
    }
  }
}

}  // namespace rr
}  // namespace lk
