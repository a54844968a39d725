// LayerNorm forward / backward.
//
// Forward (rowfuse/ops.py:248-275; Liger LK/ops/layer_norm.py:169-227):
//   mu = mean(x), r = 1/sqrt(mean((x - mu)^2) + eps), y = (x - mu) * r * w + b,
//   per-row mean and r cached in fp32.  One CTA per row, the row in registers, sums shifted
//   by the row's first element so one CTA reduction (a single barrier) gives the centred
//   variance without the E[x^2] - mean^2 cancellation; packed fp32x2 math.
// Backward (rowfuse/ops.py:278-311; LK/ops/layer_norm.py:230-304):
//   xt = (x - mu) r, gy = dy w, dx = r (gy - (xt . gy / n) xt - sum(gy) / n),
//   dw = sum_rows dy xt, db = sum_rows dy.  Persistent CTAs over contiguous row ranges,
//   rows prefetched `slots` ahead into a shared-memory ring by 1D bulk copies (issued by
//   thread 0 after the row barrier), both row reductions in one CTA barrier, dw/db
//   partials in registers -> one partial row each per CTA -> fixed-order column sums
//   (rowfuse's _tree_sum role, ops.py:138-152): bitwise deterministic for a given grid.
#include "norm_cta.cuh"

namespace lk {
namespace ln {

using rc::cta_sum;
using rc::ldg_stream;

// Two sums over the CTA's warps at once (one barrier); sh holds >= 2 x 64 floats.
__device__ __forceinline__ float2 cta_sum2(float a, float b, float* sh, int par) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) { sh[par * 64 + warp] = a; sh[par * 64 + 32 + warp] = b; }
  __syncthreads();
  float ta = lane < nw ? sh[par * 64 + lane] : 0.f;
  float tb = lane < nw ? sh[par * 64 + 32 + lane] : 0.f;
  return make_float2(warp_sum(ta), warp_sum(tb));  // fixed trees: deterministic
}

template <typename T, int VPT>
__global__ void __launch_bounds__(256) layernorm_fwd_cta(const T* __restrict__ x, const T* __restrict__ w,
                                                         const T* __restrict__ b, T* __restrict__ y,
                                                         float* __restrict__ mean, float* __restrict__ rstd,
                                                         int rows, int cols, float eps) {
  using P = ring::Pairs<T>;
  constexpr int NP = P::NP, NV = 16 / sizeof(T);
  __shared__ float sh[128];
  const int nvec = cols / NV, row = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const T* xr = x + (int64_t)row * cols;
  float2 f[VPT][NP];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    P::unpack(v < nvec ? ldg_stream(xr + v * NV) : make_uint4(0, 0, 0, 0), f[k]);
  }
  // shifted sums around K = x[row, 0] (one broadcast L1 load): var = (S2 - S1^2 / n) / n with
  // S1 = sum(x - K), S2 = sum((x - K)^2) -- one CTA reduction of two values, and no
  // E[x^2] - mean^2 cancellation because K sits inside the row's distribution
  const float K = to_f<T>(xr[0]);
  const float2 nk = make_float2(-K, -K);
  float2 s1 = make_float2(0.f, 0.f), s2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    if (tid + k * nt >= nvec) continue;
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      const float2 d = __fadd2_rn(f[k][e], nk);
      s1 = __fadd2_rn(s1, d);
      s2 = __ffma2_rn(d, d, s2);
    }
  }
  const float2 tot = cta_sum2(s1.x + s1.y, s2.x + s2.y, reinterpret_cast<float*>(sh), 0);
  const float dm = tot.x / (float)cols;
  const float mu = K + dm;
  const float m2 = fmaxf(tot.y - tot.x * dm, 0.f);
  const float r = rsqrtf(m2 / (float)cols + eps);
  if (tid == 0) { mean[row] = mu; rstd[row] = r; }
  const float2 nmu = make_float2(-mu, -mu), r2 = make_float2(r, r);
  T* yr = y + (int64_t)row * cols;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    if (v < nvec) {
      float2 wv[NP], bv[NP];
      P::unpack(__ldg(reinterpret_cast<const uint4*>(w) + v), wv);
      if (b) P::unpack(__ldg(reinterpret_cast<const uint4*>(b) + v), bv);
#pragma unroll
      for (int e = 0; e < NP; ++e) {
        const float2 t = __fmul2_rn(__fmul2_rn(__fadd2_rn(f[k][e], nmu), r2), wv[e]);
        f[k][e] = b ? __fadd2_rn(t, bv[e]) : t;
      }
      ring::stg128(yr + v * NV, P::pack(f[k]));
    }
  }
}

template <typename T, int VPT>
__global__ void __launch_bounds__(256) layernorm_bwd_cta(const T* dy, const T* __restrict__ x,
                                                         const T* __restrict__ w, const float* __restrict__ mean,
                                                         const float* __restrict__ rstd, T* dx,
                                                         float* __restrict__ dw_part, float* __restrict__ db_part,
                                                         int rows, int cols, int slots) {
  rc::allow_dependents();
  using P = ring::Pairs<T>;
  constexpr int NP = P::NP, NV = 16 / sizeof(T);
  __shared__ float sh[128];
  __shared__ uint64_t full[8];
  extern __shared__ __align__(128) uint8_t ring_sm[];
  const int nvec = cols / NV, tid = threadIdx.x, nt = blockDim.x;
  const uint32_t rb = (uint32_t)cols * sizeof(T);
  const int per = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float2 aw[VPT][NP], ab[VPT][NP], wv[VPT][NP];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    if (v < nvec) P::unpack(__ldg(reinterpret_cast<const uint4*>(w) + v), wv[k]);
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      aw[k][e] = ab[k][e] = make_float2(0.f, 0.f);
      if (v >= nvec) wv[k][e] = make_float2(0.f, 0.f);
    }
  }
  auto issue = [&](int row, int slot) {  // thread 0 only: dy row and x row into one ring slot
    uint8_t* st = ring_sm + (size_t)slot * 2 * rb;
    ring::expect_tx(&full[slot], 2 * rb);
    ring::bulk_g2s(st, dy + (int64_t)row * cols, rb, &full[slot]);
    ring::bulk_g2s(st + rb, x + (int64_t)row * cols, rb, &full[slot]);
  };
  if (tid == 0) {
    for (int q = 0; q < slots; ++q) ring::mbar_init(&full[q], 1);
    ring::fence_init();
    for (int q = 0; q < slots && r0 + q < r1; ++q) issue(r0 + q, q);
  }
  __syncthreads();
  const uint32_t base = ring::s_u32(ring_sm);
  ring::Cursor cur(slots);
  int par = 0;
  for (int row = r0; row < r1; ++row, par ^= 1, cur.next()) {
    const float mu = mean[row], r = rstd[row];
    const float2 nmu = make_float2(-mu, -mu), r2 = make_float2(r, r);
    const uint32_t st = base + (uint32_t)cur.s * 2u * rb;
    ring::wait(&full[cur.s], cur.phase);
    float2 xt[VPT][NP], gy[VPT][NP];
    float2 pj = make_float2(0.f, 0.f), sf = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int v = tid + k * nt;
      const bool in = v < nvec;
      float2 g[NP], xv[NP];
      P::unpack(in ? ring::lds128(st + (uint32_t)v * 16u) : make_uint4(0, 0, 0, 0), g);
      P::unpack(in ? ring::lds128(st + rb + (uint32_t)v * 16u) : make_uint4(0, 0, 0, 0), xv);
#pragma unroll
      for (int e = 0; e < NP; ++e) {
        xt[k][e] = in ? __fmul2_rn(__fadd2_rn(xv[e], nmu), r2) : make_float2(0.f, 0.f);
        gy[k][e] = __fmul2_rn(g[e], wv[k][e]);
        pj = __ffma2_rn(xt[k][e], gy[k][e], pj);
        sf = __fadd2_rn(sf, gy[k][e]);
        aw[k][e] = __ffma2_rn(g[e], xt[k][e], aw[k][e]);
        ab[k][e] = __fadd2_rn(ab[k][e], g[e]);
      }
    }
    const float2 t = cta_sum2(pj.x + pj.y, sf.x + sf.y, sh, par);
    // every thread is past its reads of this slot (cta_sum2's barrier): refill it
    if (tid == 0 && row + slots < r1) issue(row + slots, cur.s);
    const float proj = t.x / (float)cols, shift = t.y / (float)cols;
    const float2 np2 = make_float2(-proj, -proj), ns2 = make_float2(-shift, -shift);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int v = tid + k * nt;
      if (v < nvec) {
        float2 o[NP];
#pragma unroll
        for (int e = 0; e < NP; ++e)
          o[e] = __fmul2_rn(__fadd2_rn(__ffma2_rn(np2, xt[k][e], gy[k][e]), ns2), r2);
        ring::stg128(dx + (int64_t)row * cols + v * NV, P::pack(o));
      }
    }
  }
  float* pw = dw_part + (int64_t)blockIdx.x * cols;
  float* pb = db_part ? db_part + (int64_t)blockIdx.x * cols : nullptr;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int v = tid + k * nt;
    if (v < nvec) {
#pragma unroll
      for (int e = 0; e < NP; e += 2) {
        reinterpret_cast<float4*>(pw + v * NV)[e / 2] =
            make_float4(aw[k][e].x, aw[k][e].y, aw[k][e + 1].x, aw[k][e + 1].y);
        if (pb)
          reinterpret_cast<float4*>(pb + v * NV)[e / 2] =
              make_float4(ab[k][e].x, ab[k][e].y, ab[k][e + 1].x, ab[k][e + 1].y);
      }
    }
  }
}

// Generic fallbacks (any width, any alignment; Liger's Triton LayerNorm takes any hidden size):
// scalar loads, the row re-read from L2 in the second pass.  Forward: one 256-thread CTA per
// row.  Backward: persistent CTAs over row ranges; each thread owns columns tid, tid + 256, ...
// of its CTA's dgamma / dbeta partial row in global memory (no races), summed by the same
// fixed-order column-sum launch as the fast path.
template <typename T>
__global__ void __launch_bounds__(256) layernorm_fwd_generic(const T* __restrict__ x, const T* __restrict__ w,
                                                             const T* __restrict__ b, T* __restrict__ y,
                                                             float* __restrict__ mean, float* __restrict__ rstd,
                                                             int cols, float eps) {
  __shared__ float sh[128];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * cols;
  const float K = to_f<T>(xr[0]);
  float s1 = 0.f, s2 = 0.f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float d = to_f<T>(xr[c]) - K;
    s1 += d;
    s2 = fmaf(d, d, s2);
  }
  const float2 tot = cta_sum2(s1, s2, sh, 0);
  const float dm = tot.x / (float)cols, mu = K + dm;
  const float r = rsqrtf(fmaxf(tot.y - tot.x * dm, 0.f) / (float)cols + eps);
  if (threadIdx.x == 0) { mean[row] = mu; rstd[row] = r; }
  T* yr = y + row * cols;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float v = (to_f<T>(xr[c]) - mu) * r * to_f<T>(w[c]);
    yr[c] = from_f<T>(b ? v + to_f<T>(b[c]) : v);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) layernorm_bwd_generic(const T* dy, const T* __restrict__ x,
                                                             const T* __restrict__ w, const float* __restrict__ mean,
                                                             const float* __restrict__ rstd, T* dx,
                                                             float* __restrict__ dw_part, float* __restrict__ db_part,
                                                             int rows, int cols) {
  rc::allow_dependents();
  __shared__ float sh[128];
  const int per = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float* pw = dw_part + (int64_t)blockIdx.x * cols;
  float* pb = db_part ? db_part + (int64_t)blockIdx.x * cols : nullptr;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    pw[c] = 0.f;
    if (pb) pb[c] = 0.f;
  }
  int par = 0;
  for (int row = r0; row < r1; ++row, par ^= 1) {
    const float mu = mean[row], r = rstd[row];
    const T* xr = x + (int64_t)row * cols;
    const T* gr = dy + (int64_t)row * cols;
    float pj = 0.f, sf = 0.f;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      const float g = to_f<T>(gr[c]), xt = (to_f<T>(xr[c]) - mu) * r, gy = g * to_f<T>(w[c]);
      pj = fmaf(xt, gy, pj);
      sf += gy;
      pw[c] = fmaf(g, xt, pw[c]);
      if (pb) pb[c] += g;
    }
    const float2 t = cta_sum2(pj, sf, sh, par);
    const float proj = t.x / (float)cols, shift = t.y / (float)cols;
    T* dxr = dx + (int64_t)row * cols;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {  // dx may alias dy: read before write
      const float xt = (to_f<T>(xr[c]) - mu) * r, gy = to_f<T>(gr[c]) * to_f<T>(w[c]);
      dxr[c] = from_f<T>((gy - proj * xt - shift) * r);
    }
  }
}

static int vpt_for(int64_t nvec, int* threads, int target = 256) {
  int v = 1;
  while (v < 8 && (nvec + v - 1) / v > target) v *= 2;
  if ((nvec + v - 1) / v > 256) return 0;
  *threads = (int)(((nvec + v - 1) / v + 31) / 32 * 32);
  return v;
}
static int64_t bwd_grid(int64_t rows) { return std::max<int64_t>(1, std::min<int64_t>(rows, 8 * (int64_t)sm_count())); }

}  // namespace ln

// defined in norm.cu
int launch_colsum_partials(const float* p0, void* o0, const float* p1, void* o1, int64_t g, int64_t cols, int dtype,
                           cudaStream_t st);

}  // namespace lk

using namespace lk;

#define LK_LN_VPT(vpt, VPT, ...)                            \
  switch (vpt) {                                            \
    case 1: { constexpr int VPT = 1; __VA_ARGS__; break; }  \
    case 2: { constexpr int VPT = 2; __VA_ARGS__; break; }  \
    case 4: { constexpr int VPT = 4; __VA_ARGS__; break; }  \
    default: { constexpr int VPT = 8; __VA_ARGS__; break; } \
  }

extern "C" int lk_layernorm_fwd(const void* x, const void* weight, const void* bias, void* y, float* mean,
                                float* rstd, int64_t rows, int64_t cols, float eps, int dtype, void* stream) {
  LK_REQUIRE(rows >= 0 && cols >= 1, LK_SIZE_MISMATCH, "rows >= 0 and cols >= 1 required");
  if (rows == 0) return LK_OK;
  LK_REQUIRE(x && weight && y && mean && rstd, LK_INVALID_ARGUMENT, "null pointer");
  LK_REQUIRE(rows <= 0x7fffffff, LK_SIZE_MISMATCH, "too many rows");
  LK_REQUIRE(cols <= 0x7fffffff, LK_SIZE_MISMATCH, "hidden size too large");
  const int64_t nv = dtype == LK_F32 ? 4 : 8;
  const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(weight) |
                         reinterpret_cast<uintptr_t>(bias) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  int threads = 0;
  const int vpt = cols % nv == 0 && aligned ? ln::vpt_for(cols / nv, &threads, 128) : 0;
  cudaStream_t st = as_stream(stream);
  if (vpt == 0) {  // ragged / unaligned / wider than the register kernel
    LK_DISPATCH_FLOAT(dtype, T, {
      ln::layernorm_fwd_generic<T><<<(unsigned)rows, 256, 0, st>>>(
          static_cast<const T*>(x), static_cast<const T*>(weight), static_cast<const T*>(bias), static_cast<T*>(y),
          mean, rstd, (int)cols, eps);
    });
    return check_launch("layernorm_fwd_generic");
  }
  LK_DISPATCH_FLOAT(dtype, T, {
    LK_LN_VPT(vpt, VPT, {
      ln::layernorm_fwd_cta<T, VPT><<<(unsigned)rows, threads, 0, st>>>(
          static_cast<const T*>(x), static_cast<const T*>(weight), static_cast<const T*>(bias), static_cast<T*>(y),
          mean, rstd, (int)rows, (int)cols, eps);
    });
  });
  return check_launch("layernorm_fwd_cta");
}

extern "C" size_t lk_layernorm_bwd_workspace_bytes(int64_t rows, int64_t cols) {
  return (size_t)2 * ln::bwd_grid(rows) * (size_t)cols * sizeof(float) + 256;
}

extern "C" int lk_layernorm_bwd(const void* dy, const void* x, const void* weight, const float* mean,
                                const float* rstd, void* dx, void* dw, void* db, int64_t rows, int64_t cols,
                                int dtype, void* workspace, size_t workspace_bytes, void* stream) {
  LK_REQUIRE(rows >= 0 && cols >= 1, LK_SIZE_MISMATCH, "rows >= 0 and cols >= 1 required");
  LK_REQUIRE(rows <= 0x7fffffff, LK_SIZE_MISMATCH, "too many rows");
  LK_REQUIRE(weight && dw, LK_INVALID_ARGUMENT, "null weight / dw");
  LK_REQUIRE(workspace && workspace_bytes >= lk_layernorm_bwd_workspace_bytes(rows, cols), LK_INVALID_ARGUMENT,
             "workspace too small");
  LK_REQUIRE(rows == 0 || (dy && x && mean && rstd && dx), LK_INVALID_ARGUMENT, "null pointer");
  LK_REQUIRE(cols <= 0x7fffffff, LK_SIZE_MISMATCH, "hidden size too large");
  const int64_t nv = dtype == LK_F32 ? 4 : 8;
  cudaStream_t st = as_stream(stream);
  float* pw = static_cast<float*>(workspace);
  const int64_t gmax = ln::bwd_grid(rows);
  float* pb = pw + gmax * cols;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(x) |
                         reinterpret_cast<uintptr_t>(weight) | reinterpret_cast<uintptr_t>(dx)) & 15) == 0;
  int threads = 0;
  int vpt = cols % nv == 0 && aligned ? ln::vpt_for(cols / nv, &threads) : 0;
  // the TMA ring needs >= 2 slots of (dy, x) rows in <= 200 KB of shared memory
  if (vpt && 2 * 2 * cols * (dtype == LK_F32 ? 4 : 2) > 200 * 1024) vpt = 0;
  int64_t grid = 1;
  if (rows == 0) {
    LK_CUDA(cudaMemsetAsync(pw, 0, (size_t)2 * gmax * cols * sizeof(float), st));
  } else if (vpt == 0) {  // ragged / unaligned / wide rows
    grid = std::max<int64_t>(1, std::min<int64_t>({rows, gmax, 4 * (int64_t)sm_count()}));
    LK_DISPATCH_FLOAT(dtype, T, {
      ln::layernorm_bwd_generic<T><<<(unsigned)grid, 256, 0, st>>>(
          static_cast<const T*>(dy), static_cast<const T*>(x), static_cast<const T*>(weight), mean, rstd,
          static_cast<T*>(dx), pw, db ? pb : nullptr, (int)rows, (int)cols);
    });
    int rc = check_launch("layernorm_bwd_generic");
    if (rc) return rc;
  } else {
    LK_DISPATCH_FLOAT(dtype, T, {
      LK_LN_VPT(vpt, VPT, {
        auto kern = ln::layernorm_bwd_cta<T, VPT>;
        const int64_t rbytes = cols * (int64_t)sizeof(T);
        const int slots = (int)std::max<int64_t>(2, std::min<int64_t>(3, (96 * 1024) / (2 * rbytes)));
        const int smem = (int)(slots * 2 * rbytes);
        LK_CUDA(ensure_smem(reinterpret_cast<const void*>(kern), smem));
        int per_sm = 0;
        LK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
        grid = std::max<int64_t>(1, std::min<int64_t>({rows, gmax, (int64_t)std::max(1, per_sm) * sm_count()}));
        kern<<<(unsigned)grid, threads, smem, st>>>(static_cast<const T*>(dy), static_cast<const T*>(x),
                                                    static_cast<const T*>(weight), mean, rstd, static_cast<T*>(dx), pw,
                                                    db ? pb : nullptr, (int)rows, (int)cols, slots);
      });
    });
    int rc = check_launch("layernorm_bwd_cta");
    if (rc) return rc;
  }
  return launch_colsum_partials(pw, dw, db ? pb : nullptr, db, grid, cols, dtype, st);
}
