// Shared-memory TMA ring primitives for the persistent bandwidth kernels.
//
// A persistent CTA = one producer warp + NC consumer warps.  The producer streams
// row-sized (RMSNorm) or 16 KB (cross entropy) pieces of HBM into a ring of S
// shared-memory stages with 1D bulk copies (cp.async.bulk ... complete_tx), so
// the copy engine keeps ~S stages of loads in flight per SM while the consumer
// warps reduce and write.  full[s] completes when stage s has landed; empty[s]
// completes when its consumers are done with it.
#pragma once
#include "common.cuh"
#include <type_traits>

namespace lk {
namespace ring {

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(s_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
// 32-bit shared-window address forms (hot consumer loops: no generic<->shared conversions)
__device__ __forceinline__ void arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void wait(uint32_t b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  } while (!done);
}
// Release a ring stage right after loading from it (before the loaded registers are used).
// A plain `mbarrier.arrive` after the ld.shared is NOT enough in practice: the SYNCS arrive
// can take effect while the warp's LDS are still queued behind its global stores, the
// producer then refills the stage, and the late LDS read the NEXT piece (measured on B200: a
// few 256-column stretches per ~20k FLCE finalize rows differed run to run;
// scripts/determinism_stage.py, profiles/r02/ring_release_race.md).  The arrive here
// consumes `dep`, an OR of one register of every loaded vector (an LDS.128 completes for the
// whole warp at once, so one register per load instruction carries the scoreboard wait), so
// the warp cannot issue it before all of its loads have returned.  `min(dep, 0) + bar` keeps
// the address equal to `bar` (checked in the SASS: VIMNMX.U32 feeding SYNCS.ARRIVE).
// Called by every lane; lane 0 arrives.
template <int K>
__device__ __forceinline__ void release_after_loads(uint32_t bar, const uint4 (&raw)[K], int lane) {
  uint32_t dep = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) dep |= raw[k].x;
  __syncwarp();
  if (lane == 0)
    asm volatile(
        "{\n\t.reg .b32 t;\n\tmin.u32 t, %1, 0;\n\tadd.u32 t, t, %0;\n\t"
        "mbarrier.arrive.shared::cta.b64 _, [t];\n\t}" ::"r"(bar), "r"(dep)
        : "memory");
}
// global -> shared 1D bulk copy, completion counted on `bar` (bytes multiple of 16).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(bar))
      : "memory");
}
// Named barrier over the consumer warps only (the producer never joins).
__device__ __forceinline__ void consumers_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(s_u32(p)));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {  // 32-bit shared-window address
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__host__ __device__ inline uint32_t pad128(uint64_t b) { return (uint32_t)((b + 127) / 128 * 128); }

template <typename T>
__device__ __forceinline__ void unpack(const uint4& raw, float (&v)[16 / sizeof(T)]) {
  const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
  for (int i = 0; i < (int)(16 / sizeof(T)); ++i) v[i] = to_f<T>(e[i]);
}
template <typename T>
__device__ __forceinline__ uint4 pack(const float (&v)[16 / sizeof(T)]) {
  uint4 raw;
  T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
  for (int i = 0; i < (int)(16 / sizeof(T)); ++i) e[i] = from_f<T>(v[i]);
  return raw;
}
// 16-byte global store that does not allocate in L1 (results are not re-read by this SM).
__device__ __forceinline__ void stg128(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// 16-byte vector <-> NP float2 pairs
template <typename T> struct Pairs;
template <> struct Pairs<__nv_bfloat16> {
  static constexpr int NP = 4;
  static __device__ __forceinline__ void unpack(const uint4& r, float2 (&p)[NP]) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xffff0000u));
  }
  static __device__ __forceinline__ uint4 pack(const float2 (&p)[NP]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(p[i].x, p[i].y);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <> struct Pairs<__half> {
  static constexpr int NP = 4;
  static __device__ __forceinline__ void unpack(const uint4& r, float2 (&p)[NP]) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
  }
  static __device__ __forceinline__ uint4 pack(const float2 (&p)[NP]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = __floats2half2_rn(p[i].x, p[i].y);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <> struct Pairs<float> {
  static constexpr int NP = 2;
  static __device__ __forceinline__ void unpack(const uint4& r, float2 (&p)[NP]) {
    p[0] = make_float2(__uint_as_float(r.x), __uint_as_float(r.y));
    p[1] = make_float2(__uint_as_float(r.z), __uint_as_float(r.w));
  }
  static __device__ __forceinline__ uint4 pack(const float2 (&p)[NP]) {
    return make_uint4(__float_as_uint(p[0].x), __float_as_uint(p[0].y), __float_as_uint(p[1].x),
                      __float_as_uint(p[1].y));
  }
};

// round each lane of a float2 through T (a cast to the storage dtype and back)
template <typename T>
__device__ __forceinline__ float2 round2(float2 v) {
  if constexpr (sizeof(T) == 4) {
    return v;
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
    const uint32_t u = *reinterpret_cast<uint32_t*>(&h);
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
  } else {
    return __half22float2(__floats2half2_rn(v.x, v.y));
  }
}

// Ring position: stage index and the parity of the number of completed passes over the
// ring (incremental -- a 64-bit `q % stages` would cost a ~70-instruction division).
struct Cursor {
  int s = 0, n;
  uint32_t phase = 0;
  bool wrapped = false;
  __device__ explicit Cursor(int stages) : n(stages) {}
  __device__ __forceinline__ void next() {
    if (++s == n) { s = 0; phase ^= 1u; wrapped = true; }
  }
};

constexpr int MAX_SMEM = 227 * 1024;

}  // namespace ring
}  // namespace lk
