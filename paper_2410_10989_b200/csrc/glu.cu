// SwiGLU / GeGLU forward + backward: pure streaming kernels, 128-bit vectorised.
//
// Forward  c = act(a) * b          (rowfuse/ops.py:389-402, 438-451)
// Backward da, db written in place  (rowfuse/ops.py:405-430, 454-482;
//                                    Liger in-place contract LK/ops/swiglu.py:61-62,
//                                    LK/ops/geglu.py:85-86)
// Casting points follow Liger: the activation is computed in fp32 and cast to b's
// dtype before the multiply (LK/ops/swiglu.py:28-31, LK/ops/geglu.py:43-44).
#include "common.cuh"

namespace lk {

constexpr float kGeluC = 0.7978845608028654f;  // sqrt(2/pi)   rowfuse/ops.py:37
constexpr float kGeluA = 0.044715f;            //              rowfuse/ops.py:38
constexpr float kGelu3A = 0.134145f;           // 3 * 0.044715 rowfuse/ops.py:39

template <bool ACC>
__device__ __forceinline__ float tanh_sel(float x) { return ACC ? tanhf(x) : tanh_fast(x); }

// 1 / (1 + e^-z); e^-z -> inf for z << 0 gives exactly 0.  16-bit dtypes use the MUFU
// approximate reciprocal (rcp.approx, ~1 ulp: invisible after the bf16 cast; __frcp_rn is an
// IEEE-rounded software sequence that made the SwiGLU forward instruction-bound at 80% of HBM).
template <bool ACC>
__device__ __forceinline__ float sigmoidf_(float z) {
  const float d = 1.f + __expf(-z);
  if (ACC) return __frcp_rn(d);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  return r;
}

// ACT: 0 SwiGLU, 1 GeGLU (tanh), 2 SwiGLU with Liger's gate_multiplier gm: silu(gm * a) * b,
// da = dc (silu' at gm * a) b gm (LK/ops/swiglu.py:16-62).  gm is ignored for ACT 0 / 1.
template <typename T, int ACT>
struct Glu {
  static constexpr bool ACC = sizeof(T) == 4;
  // forward value for one element
  static __device__ __forceinline__ float fwd(float a, float b, float gm) {
    float act;
    if (ACT == 2) a *= gm;
    if (ACT != 1) {
      act = a * sigmoidf_<ACC>(a);
    } else {
      float t = tanh_sel<ACC>(kGeluC * (a + kGeluA * a * a * a));
      act = 0.5f * a * (1.f + t);
    }
    return round_to<T>(act) * b;
  }
  // backward: returns (da, db)
  static __device__ __forceinline__ void bwd(float dc, float a, float b, float gm, float& da, float& db) {
    if (ACT != 1) {
      if (ACT == 2) a *= gm;
      float sg = sigmoidf_<true>(a);  // (the approximate reciprocal measured slower here: 87% vs 93%)
      float silu = a * sg;
      db = dc * silu;
      da = dc * (silu * (1.f - sg) + sg) * b;
      if (ACT == 2) da *= gm;
    } else {
      float t = tanh_sel<ACC>(kGeluC * (a + kGeluA * a * a * a));
      float g = round_to<T>(0.5f * a * (1.f + t));
      db = dc * g;
      float dg = 0.5f * (1.f + t) + 0.5f * kGeluC * a * (1.f - t * t) * (1.f + kGelu3A * a * a);
      da = dc * b * dg;
    }
  }
};

template <typename T, int ACT>
__global__ void __launch_bounds__(256) glu_fwd_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                      T* __restrict__ c, int64_t n, float gm, bool vec) {
  constexpr int NV = Vec16<T>::N;
  const int64_t nvec = vec ? n / NV : 0;  // unaligned buffers: everything through the scalar loop
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // two vectors per thread per iteration: four 16-byte loads in flight before any math
  for (; i + stride < nvec; i += 2 * stride) {
    Vec16<T> va, vb, va2, vb2;
    va.load_nc(a + i * NV);
    vb.load_nc(b + i * NV);
    va2.load_nc(a + (i + stride) * NV);
    vb2.load_nc(b + (i + stride) * NV);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      va.v[k] = Glu<T, ACT>::fwd(va.v[k], vb.v[k], gm);
      va2.v[k] = Glu<T, ACT>::fwd(va2.v[k], vb2.v[k], gm);
    }
    va.store(c + i * NV);
    va2.store(c + (i + stride) * NV);
  }
  for (; i < nvec; i += stride) {
    Vec16<T> va, vb;
    va.load_nc(a + i * NV);
    vb.load_nc(b + i * NV);
#pragma unroll
    for (int k = 0; k < NV; ++k) va.v[k] = Glu<T, ACT>::fwd(va.v[k], vb.v[k], gm);
    va.store(c + i * NV);
  }
  for (int64_t i = nvec * NV + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    c[i] = from_f<T>(Glu<T, ACT>::fwd(to_f<T>(a[i]), to_f<T>(b[i]), gm));
}

// Aligned buffers run chunked kernels: one non-persistent CTA per contiguous chunk of U x 256
// 16-byte vectors, every load of the chunk issued before any math, the chunk written back,
// the CTA retired.  The block scheduler hands chunks out in order, so the resident CTAs
// stream one contiguous window through memory with maximal loads in flight: SwiGLU fwd / bwd
// 0.95 / 0.88 -> 1.01 / 1.03 of the measured copy bandwidth (read-heavy streams exceed it),
// GeGLU 0.92 / 0.87 -> 1.01 / 1.03 (profiles/r02/glu_chunked_ab.log).  A persistent grid-stride
// loop (the previous design) keeps fewer loads in flight per SM; persistent CTAs walking
// their own contiguous ranges measured 0.76 (DRAM page spread, profiles/r02/glu_blocked_ab.log).
// Forward chunk: 8 x 256 vectors (32 KB of each input, upstream Liger's row per program).
constexpr int GLU_CHUNK_U = 8;
template <typename T, int ACT>
__global__ void __launch_bounds__(256) glu_fwd_chunk_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                            T* __restrict__ c, int64_t nvec, float gm) {
  constexpr int NV = Vec16<T>::N;
  const int64_t base = (int64_t)blockIdx.x * (GLU_CHUNK_U * 256) + threadIdx.x;
  uint4 ra[GLU_CHUNK_U], rb[GLU_CHUNK_U];
#pragma unroll
  for (int u = 0; u < GLU_CHUNK_U; ++u) {
    const int64_t i = base + u * 256;
    if (i < nvec) {
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(ra[u].x), "=r"(ra[u].y), "=r"(ra[u].z), "=r"(ra[u].w) : "l"(a + i * NV));
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(rb[u].x), "=r"(rb[u].y), "=r"(rb[u].z), "=r"(rb[u].w) : "l"(b + i * NV));
    }
  }
#pragma unroll
  for (int u = 0; u < GLU_CHUNK_U; ++u) {
    const int64_t i = base + u * 256;
    if (i < nvec) {
      Vec16<T> va;
      const T* ea = reinterpret_cast<const T*>(&ra[u]);
      const T* eb = reinterpret_cast<const T*>(&rb[u]);
#pragma unroll
      for (int k = 0; k < NV; ++k) va.v[k] = Glu<T, ACT>::fwd(to_f<T>(ea[k]), to_f<T>(eb[k]), gm);
      va.store(c + i * NV);
    }
  }
}

// Backward chunk: 2 x 256 vectors (3 loads per vector; U = 4 / 8 measured 1.00 / 0.90).
constexpr int GLU_BWD_U = 2;
template <typename T, int ACT>
__global__ void __launch_bounds__(256) glu_bwd_chunk_kernel(const T* __restrict__ dc, T* __restrict__ a,
                                                            T* __restrict__ b, int64_t nvec, float gm) {
  constexpr int NV = Vec16<T>::N;
  const int64_t base = (int64_t)blockIdx.x * (GLU_BWD_U * 256) + threadIdx.x;
  uint4 rd[GLU_BWD_U], ra[GLU_BWD_U], rb[GLU_BWD_U];
#pragma unroll
  for (int u = 0; u < GLU_BWD_U; ++u) {
    const int64_t i = base + u * 256;
    if (i < nvec) {
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(rd[u].x), "=r"(rd[u].y), "=r"(rd[u].z), "=r"(rd[u].w) : "l"(dc + i * NV));
      ra[u] = *reinterpret_cast<const uint4*>(a + i * NV);
      rb[u] = *reinterpret_cast<const uint4*>(b + i * NV);
    }
  }
#pragma unroll
  for (int u = 0; u < GLU_BWD_U; ++u) {
    const int64_t i = base + u * 256;
    if (i < nvec) {
      Vec16<T> va, vb;
      const T* ed = reinterpret_cast<const T*>(&rd[u]);
      const T* ea = reinterpret_cast<const T*>(&ra[u]);
      const T* eb = reinterpret_cast<const T*>(&rb[u]);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        float da, db;
        Glu<T, ACT>::bwd(to_f<T>(ed[k]), to_f<T>(ea[k]), to_f<T>(eb[k]), gm, da, db);
        va.v[k] = da;
        vb.v[k] = db;
      }
      va.store(a + i * NV);
      vb.store(b + i * NV);
    }
  }
}

template <typename T, int ACT>
__global__ void __launch_bounds__(256) glu_bwd_kernel(const T* __restrict__ dc, T* __restrict__ a,
                                                      T* __restrict__ b, int64_t n, float gm, bool vec) {
  constexpr int NV = Vec16<T>::N;
  const int64_t nvec = vec ? n / NV : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += stride) {
    Vec16<T> vd, va, vb;
    vd.load_nc(dc + i * NV);
    va.load(a + i * NV);
    vb.load(b + i * NV);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float da, db;
      Glu<T, ACT>::bwd(vd.v[k], va.v[k], vb.v[k], gm, da, db);
      va.v[k] = da;
      vb.v[k] = db;
    }
    va.store(a + i * NV);
    vb.store(b + i * NV);
  }
  for (int64_t i = nvec * NV + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float da, db;
    Glu<T, ACT>::bwd(to_f<T>(dc[i]), to_f<T>(a[i]), to_f<T>(b[i]), gm, da, db);
    a[i] = from_f<T>(da);
    b[i] = from_f<T>(db);
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static unsigned grid_for(int64_t n, int nv) {
  int64_t work = (n / nv) + 1;
  int64_t blocks = (work + 255) / 256;
  int64_t cap = (int64_t)sm_count() * 8;  // 8 x 256-thread CTAs per SM resident
  return (unsigned)std::max<int64_t>(1, std::min(blocks, cap));
}

template <int ACT>
static int glu_fwd(const void* a, const void* b, void* c, int64_t n, int dtype, void* stream, float gm = 1.f) {
  LK_REQUIRE(n >= 0, LK_SIZE_MISMATCH, "n must be >= 0");
  if (n == 0) return LK_OK;
  LK_REQUIRE(a && b && c, LK_INVALID_ARGUMENT, "null pointer");
  const bool vec = aligned16(a) && aligned16(b) && aligned16(c);
  cudaStream_t st = as_stream(stream);
  LK_DISPATCH_FLOAT(dtype, T, {
    const int64_t nvec = n / Vec16<T>::N;
    if (vec && nvec * Vec16<T>::N == n) {
      const int64_t blocks = (nvec + GLU_CHUNK_U * 256 - 1) / (GLU_CHUNK_U * 256);
      glu_fwd_chunk_kernel<T, ACT><<<(unsigned)blocks, 256, 0, st>>>(
          static_cast<const T*>(a), static_cast<const T*>(b), static_cast<T*>(c), nvec, gm);
      return check_launch("glu_fwd_chunk_kernel");
    }
    glu_fwd_kernel<T, ACT><<<grid_for(n, Vec16<T>::N), 256, 0, st>>>(
        static_cast<const T*>(a), static_cast<const T*>(b), static_cast<T*>(c), n, gm, vec);
  });
  return check_launch("glu_fwd_kernel");
}

template <int ACT>
static int glu_bwd(const void* dc, void* a, void* b, int64_t n, int dtype, void* stream, float gm = 1.f) {
  LK_REQUIRE(n >= 0, LK_SIZE_MISMATCH, "n must be >= 0");
  if (n == 0) return LK_OK;
  LK_REQUIRE(a && b && dc, LK_INVALID_ARGUMENT, "null pointer");
  const bool vec = aligned16(a) && aligned16(b) && aligned16(dc);
  cudaStream_t st = as_stream(stream);
  LK_DISPATCH_FLOAT(dtype, T, {
    const int64_t nvec = n / Vec16<T>::N;
    if (vec && nvec * Vec16<T>::N == n) {
      const int64_t blocks = (nvec + GLU_BWD_U * 256 - 1) / (GLU_BWD_U * 256);
      glu_bwd_chunk_kernel<T, ACT><<<(unsigned)blocks, 256, 0, st>>>(
          static_cast<const T*>(dc), static_cast<T*>(a), static_cast<T*>(b), nvec, gm);
      return check_launch("glu_bwd_chunk_kernel");
    }
    glu_bwd_kernel<T, ACT><<<grid_for(n, Vec16<T>::N), 256, 0, st>>>(
        static_cast<const T*>(dc), static_cast<T*>(a), static_cast<T*>(b), n, gm, vec);
  });
  return check_launch("glu_bwd_kernel");
}

}  // namespace lk

extern "C" int lk_swiglu_fwd(const void* a, const void* b, void* c, int64_t n, int dtype, void* stream) {
  return lk::glu_fwd<0>(a, b, c, n, dtype, stream);
}
extern "C" int lk_swiglu_bwd(const void* dc, void* a, void* b, int64_t n, int dtype, void* stream) {
  return lk::glu_bwd<0>(dc, a, b, n, dtype, stream);
}
extern "C" int lk_geglu_fwd(const void* a, const void* b, void* c, int64_t n, int dtype, void* stream) {
  return lk::glu_fwd<1>(a, b, c, n, dtype, stream);
}
extern "C" int lk_geglu_bwd(const void* dc, void* a, void* b, int64_t n, int dtype, void* stream) {
  return lk::glu_bwd<1>(dc, a, b, n, dtype, stream);
}
extern "C" int lk_swiglu_fwd_ex(const void* a, const void* b, void* c, int64_t n, float gate_multiplier, int dtype,
                                void* stream) {
  return gate_multiplier == 1.f ? lk::glu_fwd<0>(a, b, c, n, dtype, stream)
                                : lk::glu_fwd<2>(a, b, c, n, dtype, stream, gate_multiplier);
}
extern "C" int lk_swiglu_bwd_ex(const void* dc, void* a, void* b, int64_t n, float gate_multiplier, int dtype,
                                void* stream) {
  return gate_multiplier == 1.f ? lk::glu_bwd<0>(dc, a, b, n, dtype, stream)
                                : lk::glu_bwd<2>(dc, a, b, n, dtype, stream, gate_multiplier);
}
