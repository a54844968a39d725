// RMSNorm high-occupancy register kernels (CTA per row group; candidate default path).
//
// Forward: one CTA (nvec / VPT threads, <= 256) per row; each thread holds VPT 16-byte
// vectors of the row in registers (non-allocating loads), so the row is read once and
// written once; the row reduction is warp shuffles + one barrier.  Small CTAs and few
// registers keep ~48 warps per SM resident, which is what overlaps one row's reduction
// with other rows' loads (the RoPE / GLU kernels reach 85-95% of HBM the same way).
//
// Backward: persistent CTAs (as many per SM as fit) over contiguous row ranges; the next
// row's (dy, x) vectors are loaded into registers while the current row is reduced and
// written (software pipelining), the dgamma partial stays in registers and is written
// once per CTA, then the fixed-order column sum (rowfuse's _tree_sum role,
// rowfuse/ops.py:138-152): bitwise deterministic for a given grid.
#pragma once
#include "ring.cuh"

namespace lk {
namespace rc {

// Programmatic dependent launch: let the column-sum grid queued behind this kernel be
// scheduled while this one runs (it waits in griddepcontrol.wait for our completion).
__device__ __forceinline__ void allow_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Sum over the CTA's warps; `sh` holds >= 2 x 32 floats (double-buffered by `par`).
// With a power-of-two warp count nw, every lane reads sh[lane % nw] and a log2(nw)-step
// butterfly finishes the sum (same fixed tree in every lane group: deterministic).
__device__ __forceinline__ float cta_sum(float v, float* sh, int par) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[par * 32 + warp] = v;
  __syncthreads();
  if ((nw & (nw - 1)) == 0) {
    float t = sh[par * 32 + (lane & (nw - 1))];
    for (int o = nw >> 1; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
  }
  float t = lane < nw ? sh[par * 32 + lane] : 0.f;
  return warp_sum(t);  // fixed tree: deterministic
}

template <typename T, typename R, int VPT>
__global__ void __launch_bounds__(256)
rmsnorm_fwd_cta(const T* __restrict__ x, const T* __restrict__ w, T* __restrict__ y, R* __restrict__ rstd,
                int rows, int cols, float eps, float offset, int mode) {
  using P = ring::Pairs<T>;
  constexpr int NP = P::NP, NV = 16 / sizeof(T);
  __shared__ float sh[64];
  const int nvec = cols / NV;
  const int row = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const T* xr = x + (int64_t)row * cols;
  uint4 raw[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    raw[k] = v < nvec ? ldg_stream(xr + v * NV) : make_uint4(0, 0, 0, 0);
  }
  float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    float2 f[NP];
    P::unpack(raw[k], f);
#pragma unroll
    for (int e = 0; e < NP; ++e) s2 = __ffma2_rn(f[e], f[e], s2);
  }
  const float r = rsqrtf(cta_sum(s2.x + s2.y, sh, 0) / (float)cols + eps);
  if (tid == 0) rstd[row] = from_f<R>(r);
  const float2 r2 = make_float2(r, r);
  constexpr bool BF16 = std::is_same<T, __nv_bfloat16>::value;
  const bool hmul = BF16 && w != nullptr && offset == 0.f && mode != LK_CAST_GEMMA;
  T* yr = y + (int64_t)row * cols;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    if (v < nvec) {
      float2 f[NP];
      P::unpack(raw[k], f);
#pragma unroll
      for (int e = 0; e < NP; ++e) f[e] = __fmul2_rn(f[e], r2);
      uint4 out;
      if (hmul) {  // y = bf16(bf16(xhat) * w): one packed bf16x2 multiply (exact fp32 product, one rounding)
        const uint4 wraw = __ldg(reinterpret_cast<const uint4*>(w) + v);
        const uint4 xb = P::pack(f);
        const uint32_t xa[4] = {xb.x, xb.y, xb.z, xb.w}, wa[4] = {wraw.x, wraw.y, wraw.z, wraw.w};
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 h = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&xa[e]),
                                     *reinterpret_cast<const __nv_bfloat162*>(&wa[e]));
          o[e] = *reinterpret_cast<uint32_t*>(&h);
        }
        out = make_uint4(o[0], o[1], o[2], o[3]);
      } else {
        float2 wv[NP];
        if (w) P::unpack(__ldg(reinterpret_cast<const uint4*>(w) + v), wv);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          if (mode != LK_CAST_GEMMA) f[e] = ring::round2<T>(f[e]);  // llama / none: xhat in x dtype
          if (w) f[e] = __fmul2_rn(f[e], __fadd2_rn(wv[e], make_float2(offset, offset)));
        }
        out = P::pack(f);
      }
      ring::stg128(yr + v * NV, out);
    }
  }
}

template <typename T, typename R, int VPT>
__global__ void __launch_bounds__(512)
rmsnorm_bwd_cta(const T* dy, const T* __restrict__ x, const T* __restrict__ w, const R* __restrict__ rstd, T* dx,
                float* __restrict__ dw_part, int rows, int cols, float offset, int mode) {
  allow_dependents();
  using P = ring::Pairs<T>;
  constexpr int NP = P::NP, NV = 16 / sizeof(T);
  __shared__ float sh[64];
  const int nvec = cols / NV;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  const bool llama = mode == LK_CAST_LLAMA;
  float2 acc[VPT][NP];
#pragma unroll
  for (int k = 0; k < VPT; ++k)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc[k][e] = make_float2(0.f, 0.f);
  uint4 gn[VPT], xn[VPT];
  auto load = [&](int row, uint4 (&g)[VPT], uint4 (&xx)[VPT]) {
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int v = tid + k * nt;
      const bool ok = row < r1 && v < nvec;
      g[k] = ok ? ldg_stream(dy + (int64_t)row * cols + v * NV) : make_uint4(0, 0, 0, 0);
      xx[k] = ok ? ldg_stream(x + (int64_t)row * cols + v * NV) : make_uint4(0, 0, 0, 0);
    }
  };
  // the thread's columns are fixed for the whole CTA: keep (offset + w) unpacked in registers
  float2 wv[VPT][NP];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    if (w && v < nvec) {
      P::unpack(__ldg(reinterpret_cast<const uint4*>(w) + v), wv[k]);
#pragma unroll
      for (int e = 0; e < NP; ++e) wv[k][e] = __fadd2_rn(wv[k][e], make_float2(offset, offset));
    } else {
#pragma unroll
      for (int e = 0; e < NP; ++e) wv[k][e] = make_float2(w ? 0.f : 1.f, w ? 0.f : 1.f);
    }
  }
  load(r0, gn, xn);
  int par = 0;
  for (int row = r0; row < r1; ++row, par ^= 1) {
    uint4 xc[VPT];
    float2 m[VPT][NP];
    const float r = to_f<R>(rstd[row]);
    const float2 r2 = make_float2(r, r);
    float2 d2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      float2 g[NP], xv[NP];
      P::unpack(gn[k], g);
      P::unpack(xn[k], xv);
      xc[k] = xn[k];
#pragma unroll
      for (int e = 0; e < NP; ++e) {
        float2 mm = __fmul2_rn(g[e], wv[k][e]);
        if (llama) mm = ring::round2<T>(mm);  // (dY * W) in x dtype (LK/ops/rms_norm.py:150-170)
        m[k][e] = mm;
        d2 = __ffma2_rn(mm, xv[e], d2);
        float2 xh = __fmul2_rn(xv[e], r2);
        if (llama) xh = ring::round2<T>(xh);
        acc[k][e] = __ffma2_rn(g[e], xh, acc[k][e]);
      }
    }
    load(row + 1, gn, xn);  // next row in flight while this one is reduced and written
    const float c = r * r * r * cta_sum(d2.x + d2.y, sh, par) / (float)cols;
    const float2 nc2 = make_float2(-c, -c);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int v = tid + k * nt;
      if (v < nvec) {
        float2 xv[NP];
        P::unpack(xc[k], xv);
#pragma unroll
        for (int e = 0; e < NP; ++e) m[k][e] = __ffma2_rn(m[k][e], r2, __fmul2_rn(xv[e], nc2));
        ring::stg128(dx + (int64_t)row * cols + v * NV, P::pack(m[k]));
      }
    }
  }
  if (!dw_part) return;
  float* pr = dw_part + (int64_t)blockIdx.x * cols;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    if (v < nvec) {
      float4* q = reinterpret_cast<float4*>(pr + v * NV);
#pragma unroll
      for (int e = 0; e < NP; e += 2) q[e / 2] = make_float4(acc[k][e].x, acc[k][e].y, acc[k][e + 1].x, acc[k][e + 1].y);
    }
  }
}

// bf16, llama casting, offset 0 (the Llama-3 configuration): m = bf16(dy * w) is exactly one
// packed bf16x2 multiply (the fp32 product of two bf16 values is exact, then one rounding --
// LK/ops/rms_norm.py:150-170), m is kept packed between the passes, and w stays packed in
// registers: ~10 instructions per element instead of ~19 for the generic-mode kernel.
//
// Loads: rows are prefetched S rows ahead into a shared-memory ring by 1D bulk copies
// (one per tensor per row, issued by thread 0 right after the row barrier, when every
// thread has consumed the slot).  Register prefetch of one row ahead left only ~32 KB in
// flight per SM and the kernel latency-bound at 58% of HBM.
template <int VPT, bool EXACT>  // EXACT: nvec == VPT * blockDim.x (no column guards)
__global__ void __launch_bounds__(VPT == 1 ? 512 : 256, VPT == 1 ? 2 : (VPT == 2 ? 3 : 1))
rmsnorm_bwd_cta_bf16_llama(const __nv_bfloat16* dy, const __nv_bfloat16* __restrict__ x,
                           const __nv_bfloat16* __restrict__ w, const float* __restrict__ rstd, __nv_bfloat16* dx,
                           float* __restrict__ dw_part, int rows, int cols, int slots) {
  allow_dependents();
  using P = ring::Pairs<__nv_bfloat16>;
  __shared__ float sh[64];
  __shared__ uint64_t full[8];
  extern __shared__ __align__(128) uint8_t ring_sm[];
  const int nvec = cols / 8;
  const uint32_t rb = (uint32_t)cols * 2u;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float2 acc[VPT][4];
  uint4 wp[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    wp[k] = v < nvec ? __ldg(reinterpret_cast<const uint4*>(w) + v) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[k][e] = make_float2(0.f, 0.f);
  }
  auto issue = [&](int row, int slot) {  // thread 0 only
    uint8_t* st = ring_sm + (size_t)slot * 2 * rb;
    ring::expect_tx(&full[slot], 2 * rb);
    ring::bulk_g2s(st, dy + (int64_t)row * cols, rb, &full[slot]);
    ring::bulk_g2s(st + rb, x + (int64_t)row * cols, rb, &full[slot]);
  };
  if (tid == 0) {
    for (int s = 0; s < slots; ++s) ring::mbar_init(&full[s], 1);
    ring::fence_init();
    for (int s = 0; s < slots && r0 + s < r1; ++s) issue(r0 + s, s);
  }
  __syncthreads();
  auto lo = [](uint32_t u) { return __uint_as_float(u << 16); };
  auto hi = [](uint32_t u) { return __uint_as_float(u & 0xffff0000u); };
  ring::Cursor cur(slots);
  int par = 0;
  const uint32_t ring_base = ring::s_u32(ring_sm);  // computed once: no per-access window math
  float r_next = r0 < r1 ? rstd[r0] : 0.f;
  for (int row = r0; row < r1; ++row, par ^= 1, cur.next()) {
    const float r = r_next;
    if (row + 1 < r1) r_next = rstd[row + 1];
    const float2 r2 = make_float2(r, r);
    const uint32_t st = ring_base + (uint32_t)cur.s * 2u * rb;
    ring::wait(&full[cur.s], cur.phase);
    uint4 xc[VPT], mp[VPT];
    float2 d2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int v = tid + k * nt;
      const bool in = EXACT || v < nvec;
      const uint4 gq = in ? ring::lds128(st + (uint32_t)v * 16u) : make_uint4(0, 0, 0, 0);
      const uint4 xq = in ? ring::lds128(st + rb + (uint32_t)v * 16u) : make_uint4(0, 0, 0, 0);
      const uint32_t ga[4] = {gq.x, gq.y, gq.z, gq.w};
      const uint32_t xa[4] = {xq.x, xq.y, xq.z, xq.w};
      const uint32_t wa[4] = {wp[k].x, wp[k].y, wp[k].z, wp[k].w};
      uint32_t ma[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 mb = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&ga[e]),
                                    *reinterpret_cast<const __nv_bfloat162*>(&wa[e]));
        ma[e] = *reinterpret_cast<uint32_t*>(&mb);
        const float2 m = make_float2(lo(ma[e]), hi(ma[e]));
        const float2 xv = make_float2(lo(xa[e]), hi(xa[e]));
        d2 = __ffma2_rn(m, xv, d2);
        const float2 xh = __fmul2_rn(xv, r2);
        __nv_bfloat162 hb = __floats2bfloat162_rn(xh.x, xh.y);  // xhat in x dtype
        const uint32_t hu = *reinterpret_cast<uint32_t*>(&hb);
        acc[k][e] = __ffma2_rn(make_float2(lo(ga[e]), hi(ga[e])), make_float2(lo(hu), hi(hu)), acc[k][e]);
      }
      mp[k] = make_uint4(ma[0], ma[1], ma[2], ma[3]);
      xc[k] = xq;
    }
    const float c = r * r * r * cta_sum(d2.x + d2.y, sh, par) / (float)cols;
    // every thread is past its pass-1 reads of this slot (cta_sum's barrier): refill it
    if (tid == 0 && row + slots < r1) issue(row + slots, cur.s);
    const float2 nc2 = make_float2(-c, -c);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int v = tid + k * nt;
      if (EXACT || v < nvec) {
        const uint32_t ma[4] = {mp[k].x, mp[k].y, mp[k].z, mp[k].w};
        const uint32_t xa[4] = {xc[k].x, xc[k].y, xc[k].z, xc[k].w};
        float2 o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          o[e] = __ffma2_rn(make_float2(lo(ma[e]), hi(ma[e])), r2,
                            __fmul2_rn(make_float2(lo(xa[e]), hi(xa[e])), nc2));
        ring::stg128(dx + (int64_t)row * cols + v * 8, P::pack(o));
      }
    }
  }
  if (!dw_part) return;
  float* pr = dw_part + (int64_t)blockIdx.x * cols;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    if (v < nvec) {
      float4* q = reinterpret_cast<float4*>(pr + v * 8);
      q[0] = make_float4(acc[k][0].x, acc[k][0].y, acc[k][1].x, acc[k][1].y);
      q[1] = make_float4(acc[k][2].x, acc[k][2].y, acc[k][3].x, acc[k][3].y);
    }
  }
}

}  // namespace rc
}  // namespace lk
