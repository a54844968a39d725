// RMSNorm forward / backward.
//
// Forward (rowfuse/ops.py:190-214; Liger casting modes LK/ops/rms_norm.py:45-112):
//   y = x * rstd * (offset + w), rstd = 1/sqrt(mean(x^2) + eps), one rstd per row cached.
// Backward (rowfuse/ops.py:217-241; LK/ops/rms_norm.py:115-210):
//   dx = rstd * m - (rstd^3 / n) * (m . x) * x,  m = dy * (offset + w)
//   dw = sum_rows dy * xhat  -- two-stage: one fp32 partial row per CTA, then a
//   fixed-order column sum.  The combine order depends only on the row count and
//   the grid, so the result is bitwise reproducible (the property rowfuse gets from
//   _tree_sum, ops.py:138-152).
//
// Register path (16-byte aligned rows, cols <= 4 x 512 vectors): the row lives in
// registers between the reduction and the write, so the forward is one read + one
// write and the backward two reads + one write.  Streaming path (any other shape):
// the row is re-read from L1/L2 for the second pass.  The backward is persistent:
// grid = 2 x SMs CTAs, contiguous row ranges per CTA.
#include "common.cuh"
#include "norm_rowstream.cuh"
#include "norm_ring.cuh"
#include "norm_cta.cuh"

namespace lk {

constexpr int NORM_MAX_THREADS = 512;

template <typename T, int KV>
struct RowRegs {
  static constexpr int NV = Vec16<T>::N;
  static __device__ __forceinline__ int64_t col(int k, int tid, int bs) { return ((int64_t)k * bs + tid) * NV; }
  static __device__ __forceinline__ void load(const T* p, int64_t cols, float (&v)[KV][NV], int tid, int bs) {
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int64_t c0 = col(k, tid, bs);
      if (c0 < cols) {
        Vec16<T> t;
        t.load(p + c0);
#pragma unroll
        for (int e = 0; e < NV; ++e) v[k][e] = t.v[e];
      } else {
#pragma unroll
        for (int e = 0; e < NV; ++e) v[k][e] = 0.f;
      }
    }
  }
  static __device__ __forceinline__ void store(T* p, int64_t cols, const float (&v)[KV][NV], int tid, int bs) {
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int64_t c0 = col(k, tid, bs);
      if (c0 < cols) {
        Vec16<T> t;
#pragma unroll
        for (int e = 0; e < NV; ++e) t.v[e] = v[k][e];
        t.store(p + c0);
      }
    }
  }
};

template <typename T>
__device__ __forceinline__ float fwd_val(float x, float r, float w, bool has_w, float offset, int mode) {
  float xh = x * r;
  if (mode != LK_CAST_GEMMA) xh = round_to<T>(xh);  // llama: cast xhat to x dtype before *w
  return has_w ? xh * (offset + w) : xh;
}

// ------------------------------------------------------------ register path
template <typename T, typename R, int KV>
__global__ void __launch_bounds__(NORM_MAX_THREADS)
rmsnorm_fwd_reg(const T* __restrict__ x, const T* __restrict__ w, T* __restrict__ y, R* __restrict__ rstd,
                int64_t rows, int64_t cols, float eps, float offset, int mode) {
  using IO = RowRegs<T, KV>;
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
    if (w) {
      float wv[KV][NV];
      IO::load(w, cols, wv, tid, bs);
#pragma unroll
      for (int k = 0; k < KV; ++k)
#pragma unroll
        for (int e = 0; e < NV; ++e) v[k][e] = fwd_val<T>(v[k][e], r, wv[k][e], true, offset, mode);
    } else {
#pragma unroll
      for (int k = 0; k < KV; ++k)
#pragma unroll
        for (int e = 0; e < NV; ++e) v[k][e] = fwd_val<T>(v[k][e], r, 0.f, false, offset, mode);
    }
    IO::store(y + row * cols, cols, v, tid, bs);
  }
}

template <typename T, typename R, int KV>
__global__ void __launch_bounds__(NORM_MAX_THREADS)
rmsnorm_bwd_reg(const T* dy, const T* __restrict__ x, const T* __restrict__ w, const R* __restrict__ rstd, T* dx,
                float* __restrict__ dw_part, int64_t rows, int64_t cols, float offset, int mode) {
  using IO = RowRegs<T, KV>;
  constexpr int NV = IO::NV;
  __shared__ float scratch[32];
  const int tid = threadIdx.x, bs = blockDim.x;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float acc[KV][NV];
#pragma unroll
  for (int k = 0; k < KV; ++k)
#pragma unroll
    for (int e = 0; e < NV; ++e) acc[k][e] = 0.f;
  for (int64_t row = r0; row < r1; ++row) {
    float g[KV][NV], xv[KV][NV];
    IO::load(dy + row * cols, cols, g, tid, bs);
    IO::load(x + row * cols, cols, xv, tid, bs);
    const float r = to_f<R>(rstd[row]);
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      Vec16<T> wt;
      const int64_t c0 = IO::col(k, tid, bs);
      if (w && c0 < cols) wt.load(w + c0);
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        float mm = w ? g[k][e] * (offset + (c0 < cols ? wt.v[e] : 0.f)) : g[k][e];
        if (mode == LK_CAST_LLAMA) mm = round_to<T>(mm);  // (dY * W) in x dtype, then fp32
        dot += mm * xv[k][e];
        float xh = xv[k][e] * r;
        if (mode == LK_CAST_LLAMA) xh = round_to<T>(xh);
        acc[k][e] += g[k][e] * xh;
        g[k][e] = mm;  // g now holds m
      }
    }
    dot = block_sum(dot, scratch);
    const float c = r * r * r * dot / (float)cols;
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int e = 0; e < NV; ++e) g[k][e] = r * g[k][e] - c * xv[k][e];
    IO::store(dx + row * cols, cols, g, tid, bs);
  }
  if (dw_part) {
    float* p = dw_part + (int64_t)blockIdx.x * cols;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int64_t c0 = IO::col(k, tid, bs);
      if (c0 < cols) {
#pragma unroll
        for (int e = 0; e < NV; e += 4)
          *reinterpret_cast<float4*>(p + c0 + e) = make_float4(acc[k][e], acc[k][e + 1], acc[k][e + 2], acc[k][e + 3]);
      }
    }
  }
}

// ----------------------------------------------------------- streaming path
template <typename T, typename R>
__global__ void __launch_bounds__(256)
rmsnorm_fwd_stream(const T* __restrict__ x, const T* __restrict__ w, T* __restrict__ y, R* __restrict__ rstd,
                   int64_t rows, int64_t cols, float eps, float offset, int mode) {
  __shared__ float scratch[32];
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const T* xr = x + row * cols;
    float ss = 0.f;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      float v = to_f<T>(xr[c]);
      ss += v * v;
    }
    ss = block_sum(ss, scratch);
    const float r = rsqrtf(ss / (float)cols + eps);
    if (threadIdx.x == 0) rstd[row] = from_f<R>(r);
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
      y[row * cols + c] = from_f<T>(fwd_val<T>(to_f<T>(xr[c]), r, w ? to_f<T>(w[c]) : 0.f, w != nullptr, offset, mode));
  }
}

template <typename T, typename R>
__global__ void __launch_bounds__(256)
rmsnorm_bwd_stream(const T* dy, const T* __restrict__ x, const T* __restrict__ w, const R* __restrict__ rstd, T* dx,
                   float* __restrict__ dw_part, int64_t rows, int64_t cols, float offset, int mode) {
  __shared__ float scratch[32];
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float* p = dw_part ? dw_part + (int64_t)blockIdx.x * cols : nullptr;
  if (p)
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) p[c] = 0.f;
  auto mval = [&](float g, int64_t c) {
    float mm = w ? g * (offset + to_f<T>(w[c])) : g;
    return mode == LK_CAST_LLAMA ? round_to<T>(mm) : mm;
  };
  for (int64_t row = r0; row < r1; ++row) {
    const T* gr = dy + row * cols;
    const T* xr = x + row * cols;
    const float r = to_f<R>(rstd[row]);
    float dot = 0.f;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) dot += mval(to_f<T>(gr[c]), c) * to_f<T>(xr[c]);
    dot = block_sum(dot, scratch);
    const float cc = r * r * r * dot / (float)cols;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const float g = to_f<T>(gr[c]), xv = to_f<T>(xr[c]);
      if (p) {
        float xh = xv * r;
        if (mode == LK_CAST_LLAMA) xh = round_to<T>(xh);
        p[c] += g * xh;
      }
      dx[row * cols + c] = from_f<T>(r * mval(g, c) - cc * xv);
    }
    __syncthreads();  // dx may alias dy: finish the row before the next row's reduction
  }
}

// dw[c] = sum_g part[g, c] in a fixed order (deterministic second stage).  A CTA owns 32
// columns (one coalesced 128-byte segment per partial row) and 32 row groups: thread
// (ty, tx) sums rows ty, ty + 32, ... of column tx with 8 independent accumulators (all of a
// thread's loads in flight at once), then the 32 group sums are added in ty order.
// (One thread per column walking ~450 partial rows serially was latency-bound at 16 us.)
template <typename T>
__global__ void __launch_bounds__(1024) colsum_partials_kernel(const float* __restrict__ p0, T* __restrict__ o0,
                                                               const float* __restrict__ p1, T* __restrict__ o1,
                                                               int64_t g, int64_t cols) {
  // launched as a programmatic dependent of the backward kernel: the launch and this
  // prologue overlap the backward's tail; the partials are read only after it completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ float red[32][33];
  const float* part = blockIdx.y ? p1 : p0;
  T* out = blockIdx.y ? o1 : o0;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c = blockIdx.x * 32 + tx;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < cols) {
    int64_t i = ty;
    for (; i + 7 * 32 < g; i += 8 * 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += part[(i + u * 32) * cols + c];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i + u * 32 < g) a[u] += part[(i + u * 32) * cols + c];
  }
  red[ty][tx] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  __syncthreads();
  if (ty == 0 && c < cols) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) s += red[k][tx];
    out[c] = from_f<T>(s);
  }
}

// Fixed-order column sums of one or two [g, cols] fp32 partial arrays (dgamma, dbeta),
// deterministic for a given g; a programmatic dependent launch of the preceding kernel.
int launch_colsum_partials(const float* p0, void* o0, const float* p1, void* o1, int64_t g, int64_t cols, int dtype,
                           cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)((cols + 31) / 32), p1 ? 2u : 1u);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LK_DISPATCH_FLOAT(dtype, T, {
    LK_CUDA(cudaLaunchKernelEx(&cfg, colsum_partials_kernel<T>, p0, static_cast<T*>(o0), p1, static_cast<T*>(o1), g,
                               cols));
  });
  return check_launch("colsum_partials_kernel");
}

struct NormCfg {
  bool reg;
  int kv;
  int block;
};

template <typename T>
static NormCfg pick_cfg(int64_t cols, std::initializer_list<const void*> ptrs) {
  constexpr int NV = Vec16<T>::N;
  bool vec = (cols % NV == 0);
  for (const void* p : ptrs)
    if (p && (reinterpret_cast<uintptr_t>(p) & 15)) vec = false;
  const int64_t units = cols / NV;
  if (!vec || units > 4 * NORM_MAX_THREADS) return {false, 0, 256};
  int kv = 1;
  while (kv < 4 && (units + kv - 1) / kv > 256) kv *= 2;
  int64_t block = (units + kv - 1) / kv;
  block = std::min<int64_t>(NORM_MAX_THREADS, std::max<int64_t>(32, (block + 31) / 32 * 32));
  return {true, kv, (int)block};
}

#define LK_KV_DISPATCH(kv, KV, ...)                            \
  switch (kv) {                                                \
    case 1: { constexpr int KV = 1; __VA_ARGS__; break; }      \
    case 2: { constexpr int KV = 2; __VA_ARGS__; break; }      \
    default: { constexpr int KV = 4; __VA_ARGS__; break; }     \
  }

static bool aligned16_all(std::initializer_list<const void*> ptrs) {
  for (const void* p : ptrs)
    if (p && (reinterpret_cast<uintptr_t>(p) & 15)) return false;
  return true;
}

// Implementation choice: CTA per row (product path); warp-per-row, generic and TMA-ring kernels
// only through the LK_PATH_NORM_IMPL test knob, so the parity tests run every path against the others.
enum { IMPL_CTA = 0, IMPL_WARP = 1, IMPL_GENERIC = 2, IMPL_RING = 3 };
static int norm_impl() { return path_knob(LK_PATH_NORM_IMPL); }

#define LK_VPT8_DISPATCH(vpt, VPT, ...)                     \
  switch (vpt) {                                            \
    case 1: { constexpr int VPT = 1; __VA_ARGS__; break; }  \
    case 2: { constexpr int VPT = 2; __VA_ARGS__; break; }  \
    case 4: { constexpr int VPT = 4; __VA_ARGS__; break; }  \
    default: { constexpr int VPT = 8; __VA_ARGS__; break; } \
  }

// vectors per thread so that a row takes <= `target` threads (VPT <= 8, <= max_threads)
static int cta_vpt(int64_t nvec, int target, int max_threads) {
  int v = 1;
  while (v < 8 && (nvec + v - 1) / v > target) v *= 2;
  return (nvec + v - 1) / v <= max_threads ? v : 0;
}

template <typename T, typename R>
static int rms_fwd_cta_launch(const T* x, const T* w, T* y, R* rstd, int64_t rows, int64_t cols, float eps,
                              float offset, int mode, cudaStream_t st) {
  constexpr int NV = Vec16<T>::N;
  if (cols % NV || !aligned16_all({x, w, y}) || rows > 0x7fffffff || rows * cols > ((int64_t)1 << 40))
    return LK_UNSUPPORTED;
  const int64_t nvec = cols / NV;
  const int vpt = cta_vpt(nvec, 128, 256);
  if (!vpt) return LK_UNSUPPORTED;
  const int threads = (int)(((nvec + vpt - 1) / vpt + 31) / 32 * 32);
  LK_VPT8_DISPATCH(vpt, VPT, {
    rc::rmsnorm_fwd_cta<T, R, VPT><<<(unsigned)rows, threads, 0, st>>>(x, w, y, rstd, (int)rows, (int)cols, eps,
                                                                       offset, mode);
  });
  return check_launch("rmsnorm_fwd_cta");
}

template <typename T, typename R>
static int rms_bwd_cta_launch(const T* dy, const T* x, const T* w, const R* rstd, T* dx, float* part,
                              int64_t rows, int64_t cols, float offset, int mode, int64_t g, cudaStream_t st,
                              int64_t* g_used) {
  constexpr int NV = Vec16<T>::N;
  if (cols % NV || !aligned16_all({dy, x, w, dx}) || rows > 0x7fffffff) return LK_UNSUPPORTED;
  const int64_t nvec = cols / NV;
  int rc = LK_OK;
  if constexpr (std::is_same<T, __nv_bfloat16>::value && std::is_same<R, float>::value) {
    if (mode == LK_CAST_LLAMA && offset == 0.f && w) {
      // 128-thread CTAs (VPT = 4 at H = 4096): 82% of HBM vs 78% with 256 threads (profiles/)
      // <= 128 threads up to VPT 4, <= 256 at VPT 8 (the launch bounds)
      const int vpt = cta_vpt(nvec, 128, 256);
      if (!vpt) return LK_UNSUPPORTED;
      const int threads = (int)(((nvec + vpt - 1) / vpt + 31) / 32 * 32);
      const int64_t rb = cols * 2;
      const int slots = (int)std::max<int64_t>(2, std::min<int64_t>(3,
                                                                    (96 * 1024) / (2 * rb)));
      const int smem = (int)(slots * 2 * rb);
      if (rb % 16 || smem > 200 * 1024) return LK_UNSUPPORTED;
      const bool exact = nvec == (int64_t)vpt * threads;
      LK_VPT8_DISPATCH(vpt, VPT, {
        auto kern = exact ? rc::rmsnorm_bwd_cta_bf16_llama<VPT, true> : rc::rmsnorm_bwd_cta_bf16_llama<VPT, false>;
        LK_CUDA(ensure_smem(reinterpret_cast<const void*>(kern), smem));
        int per_sm = 0;
        LK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
        per_sm = std::max(1, std::min(per_sm, 8));
        const unsigned grid =
            (unsigned)std::max<int64_t>(1, std::min<int64_t>({rows, g, (int64_t)per_sm * sm_count()}));
        *g_used = grid;
        kern<<<grid, threads, smem, st>>>(dy, x, w, rstd, dx, part, (int)rows, (int)cols, slots);
        rc = check_launch("rmsnorm_bwd_cta_bf16_llama");
      });
      return rc;
    }
  }
  const int vpt = cta_vpt(nvec, 256, 512);
  if (!vpt) return LK_UNSUPPORTED;
  const int threads = (int)(((nvec + vpt - 1) / vpt + 31) / 32 * 32);
  LK_VPT8_DISPATCH(vpt, VPT, {
    auto kern = rc::rmsnorm_bwd_cta<T, R, VPT>;
    int per_sm = 0;
    LK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0));
    per_sm = std::max(1, std::min(per_sm, 8));
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>({rows, g, (int64_t)per_sm * sm_count()}));
    *g_used = grid;
    kern<<<grid, threads, 0, st>>>(dy, x, w, rstd, dx, part, (int)rows, (int)cols, offset, mode);
    rc = check_launch("rmsnorm_bwd_cta");
  });
  return rc;
}

#define LK_VPT_DISPATCH(vpt, VPT, ...)                      \
  switch (vpt) {                                            \
    case 1: { constexpr int VPT = 1; __VA_ARGS__; break; }  \
    case 2: { constexpr int VPT = 2; __VA_ARGS__; break; }  \
    default: { constexpr int VPT = 4; __VA_ARGS__; break; } \
  }

// Consumer warps and vectors per thread for the ring kernels: nw*32*vpt >= nvec.
static bool ring_geometry(int64_t nvec, int* nw, int* vpt) {
  *nw = (int)std::min<int64_t>(rr::MAX_NW, std::max<int64_t>(1, (nvec + 31) / 32));
  const int64_t per = (nvec + *nw * 32 - 1) / (*nw * 32);
  if (per > 4) return false;
  *vpt = per <= 1 ? 1 : (per <= 2 ? 2 : 4);
  return true;
}

// Persistent TMA-ring RMSNorm (norm_ring.cuh).  Returns LK_UNSUPPORTED when the shape
// does not fit (row > 2048 vectors, unaligned rows, fewer than 2 stages).
template <typename T, typename R>
static int rms_fwd_ring_launch(const T* x, const T* w, T* y, R* rstd, int64_t rows, int64_t cols, float eps,
                               float offset, int mode, cudaStream_t st) {
  constexpr int NV = Vec16<T>::N;
  int nw, vpt;
  if (cols % NV || !aligned16_all({x, w, y}) || !ring_geometry(cols / NV, &nw, &vpt)) return LK_UNSUPPORTED;
  const rr::Layout one = rr::layout(cols, sizeof(T), rr::FWD_RB, 1, 0);
  int stages = (int)((ring::MAX_SMEM - one.total - 256) / (one.stage_bytes + 16));
  stages = std::min(stages, 16);
  if (stages < 2) return LK_UNSUPPORTED;
  const rr::Layout L = rr::layout(cols, sizeof(T), rr::FWD_RB, 1, stages);
  const int64_t nb = (rows + rr::FWD_RB - 1) / rr::FWD_RB;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nb, sm_count()));
  int rc = LK_OK;
  LK_VPT_DISPATCH(vpt, VPT, {
    auto kern = rr::rmsnorm_fwd_ring<T, R, VPT>;
    LK_CUDA(ensure_smem(reinterpret_cast<const void*>(kern), (int)L.total));
    kern<<<grid, (nw + 1) * 32, L.total, st>>>(x, w, y, rstd, rows, cols, eps, offset, mode, stages);
    rc = check_launch("rmsnorm_fwd_ring");
  });
  return rc;
}

template <typename T, typename R>
static int rms_bwd_ring_launch(const T* dy, const T* x, const T* w, const R* rstd, T* dx, float* part,
                               int64_t rows, int64_t cols, float offset, int mode, int64_t g, cudaStream_t st,
                               int64_t* g_used) {
  constexpr int NV = Vec16<T>::N;
  int nw, vpt;
  if (cols % NV || !aligned16_all({dy, x, w, dx}) || !ring_geometry(cols / NV, &nw, &vpt)) return LK_UNSUPPORTED;
  const rr::Layout one = rr::layout(cols, sizeof(T), rr::BWD_RB, 2, 0);
  int stages = (int)((ring::MAX_SMEM - one.total - 256) / (one.stage_bytes + 16));
  stages = std::min(stages, 16);
  if (stages < 2) return LK_UNSUPPORTED;
  const rr::Layout L = rr::layout(cols, sizeof(T), rr::BWD_RB, 2, stages);
  const int64_t nb = (rows + rr::BWD_RB - 1) / rr::BWD_RB;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>({nb, g, (int64_t)sm_count()}));
  *g_used = grid;
  int rc = LK_OK;
  LK_VPT_DISPATCH(vpt, VPT, {
    auto kern = rr::rmsnorm_bwd_ring<T, R, VPT>;
    LK_CUDA(ensure_smem(reinterpret_cast<const void*>(kern), (int)L.total));
    kern<<<grid, (nw + 1) * 32, L.total, st>>>(dy, x, w, rstd, dx, part, rows, cols, offset, mode, stages);
    rc = check_launch("rmsnorm_bwd_ring");
  });
  return rc;
}

template <typename T, typename R>
static int rms_fwd_launch(const T* x, const T* w, T* y, R* rstd, int64_t rows, int64_t cols, float eps,
                          float offset, int mode, cudaStream_t st) {
  const int impl = norm_impl();
  if (impl == IMPL_CTA) {
    int rc = rms_fwd_cta_launch<T, R>(x, w, y, rstd, rows, cols, eps, offset, mode, st);
    if (rc != LK_UNSUPPORTED) return rc;
  }
  if (impl == IMPL_CTA || impl == IMPL_RING) {
    int rc = rms_fwd_ring_launch<T, R>(x, w, y, rstd, rows, cols, eps, offset, mode, st);
    if (rc != LK_UNSUPPORTED) return rc;
  }
  const int64_t nvec = cols / Vec16<T>::N;
  if ((impl == IMPL_WARP || impl == IMPL_CTA || impl == IMPL_RING) && cols % Vec16<T>::N == 0 && aligned16_all({x, w, y}) && nvec <= 32 * 16) {
    const unsigned grid = (unsigned)((rows + 3) / 4);
    const int vpl = (int)((nvec + 31) / 32);
    auto go = [&](auto kern) -> int {
      kern<<<grid, rs::FWD_THREADS, 0, st>>>(x, w, y, rstd, rows, cols, eps, offset, mode);
      return check_launch("rmsnorm_fwd_warp");
    };
    if (vpl <= 1) return go(rs::rmsnorm_fwd_warp<T, R, 1>);
    if (vpl <= 2) return go(rs::rmsnorm_fwd_warp<T, R, 2>);
    if (vpl <= 4) return go(rs::rmsnorm_fwd_warp<T, R, 4>);
    if (vpl <= 8) return go(rs::rmsnorm_fwd_warp<T, R, 8>);
    return go(rs::rmsnorm_fwd_warp<T, R, 16>);
  }
  NormCfg c = pick_cfg<T>(cols, {x, w, y});
  unsigned grid = (unsigned)std::min<int64_t>(rows, 1 << 20);
  if (c.reg) {
    LK_KV_DISPATCH(c.kv, KV, { rmsnorm_fwd_reg<T, R, KV><<<grid, c.block, 0, st>>>(x, w, y, rstd, rows, cols, eps, offset, mode); });
  } else {
    rmsnorm_fwd_stream<T, R><<<grid, 256, 0, st>>>(x, w, y, rstd, rows, cols, eps, offset, mode);
  }
  return check_launch("rmsnorm_fwd");
}

static int64_t rms_bwd_grid(int64_t rows) {  // upper bound of the partial rows any path writes
  return std::max<int64_t>(1, std::min<int64_t>(rows, 8 * (int64_t)sm_count()));
}

template <typename T, typename R>
static int rms_bwd_launch(const T* dy, const T* x, const T* w, const R* rstd, T* dx, float* part, int64_t rows,
                          int64_t cols, float offset, int mode, int64_t g, cudaStream_t st, int64_t* g_used) {
  const int impl = norm_impl();
  if (impl == IMPL_CTA) {
    int rc = rms_bwd_cta_launch<T, R>(dy, x, w, rstd, dx, part, rows, cols, offset, mode, g, st, g_used);
    if (rc != LK_UNSUPPORTED) return rc;
  }
  if (impl == IMPL_CTA || impl == IMPL_RING) {
    int rc = rms_bwd_ring_launch<T, R>(dy, x, w, rstd, dx, part, rows, cols, offset, mode, g, st, g_used);
    if (rc != LK_UNSUPPORTED) return rc;
  }
  const int64_t nvec = cols / Vec16<T>::N;
  const int vpt = (int)((nvec + rs::BWD_THREADS - 1) / rs::BWD_THREADS);
  if ((impl == IMPL_WARP || impl == IMPL_CTA || impl == IMPL_RING) && cols % Vec16<T>::N == 0 && aligned16_all({dy, x, w, dx}) && vpt <= 2) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sm_count(), g));
    *g_used = grid;
    if (vpt <= 1)
      rs::rmsnorm_bwd_rows<T, R, 1, 4><<<grid, rs::BWD_THREADS, 0, st>>>(dy, x, w, rstd, dx, part, rows, cols, offset, mode);
    else
      rs::rmsnorm_bwd_rows<T, R, 2, 2><<<grid, rs::BWD_THREADS, 0, st>>>(dy, x, w, rstd, dx, part, rows, cols, offset, mode);
    return check_launch("rmsnorm_bwd_rows");
  }
  *g_used = g;
  NormCfg c = pick_cfg<T>(cols, {dy, x, w, dx});
  if (c.reg) {
    LK_KV_DISPATCH(c.kv, KV, { rmsnorm_bwd_reg<T, R, KV><<<(unsigned)g, c.block, 0, st>>>(dy, x, w, rstd, dx, part, rows, cols, offset, mode); });
  } else {
    rmsnorm_bwd_stream<T, R><<<(unsigned)g, 256, 0, st>>>(dy, x, w, rstd, dx, part, rows, cols, offset, mode);
  }
  return check_launch("rmsnorm_bwd");
}

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
  LK_DISPATCH_FLOAT(dtype, T, {
    const T* w = static_cast<const T*>(weight);
    if (casting_mode == LK_CAST_NONE)
      return rms_fwd_launch<T, T>(static_cast<const T*>(x), w, static_cast<T*>(y), static_cast<T*>(rstd), rows,
                                  cols, eps, offset, casting_mode, st);
    return rms_fwd_launch<T, float>(static_cast<const T*>(x), w, static_cast<T*>(y), static_cast<float*>(rstd),
                                    rows, cols, eps, offset, casting_mode, st);
  });
  return LK_OK;
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
    if (rows == 0) LK_CUDA(cudaMemsetAsync(part, 0, (size_t)g * cols * sizeof(float), st));
  }
  LK_REQUIRE(rows == 0 || (dy && x && rstd && dx), LK_INVALID_ARGUMENT, "null pointer");
  LK_DISPATCH_FLOAT(dtype, T, {
    const T* w = static_cast<const T*>(weight);
    int64_t g_used = g;
    if (rows > 0) {
      int rc = casting_mode == LK_CAST_NONE
                   ? rms_bwd_launch<T, T>(static_cast<const T*>(dy), static_cast<const T*>(x), w,
                                          static_cast<const T*>(rstd), static_cast<T*>(dx), part, rows, cols,
                                          offset, casting_mode, g, st, &g_used)
                   : rms_bwd_launch<T, float>(static_cast<const T*>(dy), static_cast<const T*>(x), w,
                                              static_cast<const float*>(rstd), static_cast<T*>(dx), part, rows,
                                              cols, offset, casting_mode, g, st, &g_used);
      if (rc) return rc;
    }
    if (part) return launch_colsum_partials(part, dw, nullptr, nullptr, g_used, cols, dtype, st);
  });
  return LK_OK;
}
