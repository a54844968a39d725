// Rotary position embedding, half-split (HF) layout, in place.
//
// rowfuse restates it as a per-row rotation from (thetas, positions)
// (rowfuse/ops.py:322-382); Liger takes precomputed cos/sin tables and rotates
// q[B, T, nq, d] and k[B, T, nk, d] in place (LK/ops/rope.py:6-112):
//   forward : y1 = x1*c - x2*s,  y2 = x2*c + x1*s
//   backward: y1 = x1*c + x2*s,  y2 = x2*c - x1*s   (sin negated, rowfuse ops.py:377-382)
// Only cos[..., :d/2] and sin[..., :d/2] are read (LK/ops/rope.py:58-68).
//
// Work item = one 16-byte vector of one half of one head of one token; q and k
// heads of a token are adjacent items, so a token's cos/sin vector is reused from
// L1 by all of its heads.
#include "common.cuh"

namespace lk {

template <typename T, typename C, bool VEC>
__global__ void __launch_bounds__(256) rope_kernel(T* __restrict__ q, T* __restrict__ k,
                                                   const C* __restrict__ cosp,
                                                   const C* __restrict__ sinp, int64_t batch,
                                                   int64_t seq, int nq, int nk, int d,
                                                   int64_t cos_batch, int backward) {
  constexpr int NV = VEC ? Vec16<T>::N : 1;
  const int half = d / 2;
  const int vph = half / NV;                // vectors per half head
  const int heads = nq + nk;
  const int64_t per_tok = (int64_t)heads * vph;
  const int64_t total = batch * seq * per_tok;
  const float sgn = backward ? -1.f : 1.f;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tok = it / per_tok;
    const int rem = (int)(it - tok * per_tok);
    const int h = rem / vph, v = rem - h * vph;
    const int64_t b = tok / seq, t = tok - b * seq;
    const int64_t crow = (cos_batch == 1 ? t : b * seq + t) * d;
    T* base = h < nq ? q + (tok * nq + h) * (int64_t)d : k + (tok * nk + (h - nq)) * (int64_t)d;
    const int i0 = v * NV;
    float x1[NV], x2[NV], c[NV], s[NV];
    if (VEC) {
      Vec16<T> a, bb;
      a.load(base + i0);
      bb.load(base + half + i0);
#pragma unroll
      for (int e = 0; e < NV; ++e) { x1[e] = a.v[e]; x2[e] = bb.v[e]; }
    } else {
      x1[0] = to_f<T>(base[i0]);
      x2[0] = to_f<T>(base[half + i0]);
    }
    if constexpr (VEC && sizeof(C) == sizeof(T)) {
      // same width as q/k: one 16-byte load each for cos and sin (rows are d-aligned)
      Vec16<C> vc, vs;
      vc.load(cosp + crow + i0);
      vs.load(sinp + crow + i0);
#pragma unroll
      for (int e = 0; e < NV; ++e) { c[e] = vc.v[e]; s[e] = sgn * vs.v[e]; }
    } else {
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        c[e] = to_f<C>(cosp[crow + i0 + e]);
        s[e] = sgn * to_f<C>(sinp[crow + i0 + e]);
      }
    }
    float y1[NV], y2[NV];
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      y1[e] = x1[e] * c[e] - x2[e] * s[e];
      y2[e] = x2[e] * c[e] + x1[e] * s[e];
    }
    if (VEC) {
      Vec16<T> a, bb;
#pragma unroll
      for (int e = 0; e < NV; ++e) { a.v[e] = y1[e]; bb.v[e] = y2[e]; }
      a.store(base + i0);
      bb.store(base + half + i0);
    } else {
      base[i0] = from_f<T>(y1[0]);
      base[half + i0] = from_f<T>(y2[0]);
    }
  }
}

// Token-major variant (the common shapes): one thread per (head, 16-byte vector) of a token,
// so the head / vector / cos-offset decomposition is computed once; q and k heads of a token
// in one CTA (cos/sin reused from L1).  One non-persistent CTA per ROPE_U consecutive tokens,
// every q/k load of the chunk issued before any rotation, the CTA retired after its stores:
// the block scheduler then streams one contiguous window through memory.  Against the
// previous semi-persistent design (each CTA walking ~10 tokens two at a time): 0.83 -> 0.89
// of HBM steady, 0.93 -> 0.97 cold, and 1.03-1.04x upstream Liger's Triton kernel at the
// kernel level (profiles/r02/rope_chunk_ab.log; 4 / 8 tokens per CTA: 0.83 / 0.57).
constexpr int ROPE_U = 2;
template <typename T, typename C>
__global__ void __launch_bounds__(1024) rope_chunk_kernel(T* __restrict__ q, T* __restrict__ k,
                                                          const C* __restrict__ cosp, const C* __restrict__ sinp,
                                                          int tokens, int seq, int nq, int nk, int d, int cos_per_tok,
                                                          int backward) {
  constexpr int NV = Vec16<T>::N;
  const int half = d / 2, vph = half / NV;
  const int h = threadIdx.x / vph, i0 = (threadIdx.x - h * vph) * NV;
  const float sgn = backward ? -1.f : 1.f;
  const int t0 = blockIdx.x * ROPE_U;
  T* const hb = h < nq ? q + (int64_t)h * d : k + (int64_t)(h - nq) * d;
  const int64_t tstride = (int64_t)(h < nq ? nq : nk) * d;
  uint4 ra[ROPE_U], rb[ROPE_U];
#pragma unroll
  for (int u = 0; u < ROPE_U; ++u) {
    if (t0 + u < tokens) {
      const T* p = hb + (int64_t)(t0 + u) * tstride;
      ra[u] = *reinterpret_cast<const uint4*>(p + i0);
      rb[u] = *reinterpret_cast<const uint4*>(p + half + i0);
    }
  }
  int pos = t0 % seq;
#pragma unroll
  for (int u = 0; u < ROPE_U; ++u) {
    const int tok = t0 + u;
    if (tok < tokens) {
      const int64_t crow = (int64_t)(cos_per_tok ? tok : pos) * d + i0;
      float c[NV], sn[NV];
      if constexpr (sizeof(C) == sizeof(T)) {
        Vec16<C> vc, vs;
        vc.load(cosp + crow);
        vs.load(sinp + crow);
#pragma unroll
        for (int e = 0; e < NV; ++e) { c[e] = vc.v[e]; sn[e] = sgn * vs.v[e]; }
      } else {
#pragma unroll
        for (int e = 0; e < NV; ++e) { c[e] = to_f<C>(cosp[crow + e]); sn[e] = sgn * to_f<C>(sinp[crow + e]); }
      }
      const T* ea = reinterpret_cast<const T*>(&ra[u]);
      const T* eb = reinterpret_cast<const T*>(&rb[u]);
      Vec16<T> a, b;
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const float x1 = to_f<T>(ea[e]), x2 = to_f<T>(eb[e]);
        a.v[e] = x1 * c[e] - x2 * sn[e];
        b.v[e] = x2 * c[e] + x1 * sn[e];
      }
      T* p = hb + (int64_t)tok * tstride;
      a.store(p + i0);
      b.store(p + half + i0);
    }
    pos = pos + 1 == seq ? 0 : pos + 1;
  }
}

template <typename T, typename C>
static int launch_rope(void* q, void* k, const void* cs, const void* sn, int64_t batch, int64_t seq,
                       int64_t nq, int64_t nk, int64_t d, int64_t cb, int backward, cudaStream_t st) {
  constexpr int NV = Vec16<T>::N;
  bool vec = ((d / 2) % NV == 0) && ((reinterpret_cast<uintptr_t>(q) & 15) == 0) &&
             ((reinterpret_cast<uintptr_t>(k) & 15) == 0);
  if (sizeof(C) == sizeof(T))  // vector cos/sin loads need 16-byte aligned tables
    vec = vec && ((reinterpret_cast<uintptr_t>(cs) & 15) == 0) && ((reinterpret_cast<uintptr_t>(sn) & 15) == 0);
  const int64_t per_tok = (nq + nk) * ((d / 2) / NV), tokens = batch * seq;
  if (vec && per_tok % 32 == 0 && per_tok <= 1024 && tokens <= 0x7fffffff) {
    const unsigned g = (unsigned)((tokens + ROPE_U - 1) / ROPE_U);
    rope_chunk_kernel<T, C><<<g, (int)per_tok, 0, st>>>(static_cast<T*>(q), static_cast<T*>(k),
                                                         static_cast<const C*>(cs), static_cast<const C*>(sn),
                                                         (int)tokens, (int)seq, (int)nq, (int)nk, (int)d,
                                                         cb == 1 ? 0 : 1, backward);
    return check_launch("rope_chunk_kernel");
  }
  const int64_t items = batch * seq * (nq + nk) * ((d / 2) / (vec ? NV : 1));
  unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, 16 * (int64_t)sm_count()));
  if (vec)
    rope_kernel<T, C, true><<<grid, 256, 0, st>>>(static_cast<T*>(q), static_cast<T*>(k),
                                                  static_cast<const C*>(cs), static_cast<const C*>(sn),
                                                  batch, seq, (int)nq, (int)nk, (int)d, cb, backward);
  else
    rope_kernel<T, C, false><<<grid, 256, 0, st>>>(static_cast<T*>(q), static_cast<T*>(k),
                                                   static_cast<const C*>(cs), static_cast<const C*>(sn),
                                                   batch, seq, (int)nq, (int)nk, (int)d, cb, backward);
  return check_launch("rope_kernel");
}

}  // namespace lk

extern "C" int lk_rope(void* q, void* k, const void* cos, const void* sin, int64_t batch, int64_t seq,
                       int64_t n_q_heads, int64_t n_kv_heads, int64_t head_dim, int64_t cos_batch,
                       int dtype, int cos_dtype, int backward, void* stream) {
  using namespace lk;
  LK_REQUIRE(head_dim >= 2 && head_dim % 2 == 0, LK_ODD_HEAD_DIM,
             "head_dim must be even and >= 2");
  LK_REQUIRE(batch >= 0 && seq >= 0 && n_q_heads >= 0 && n_kv_heads >= 0, LK_SIZE_MISMATCH,
             "negative size");
  LK_REQUIRE(cos_batch == 1 || cos_batch == batch, LK_SHAPE_MISMATCH,
             "cos/sin batch must be 1 or the q/k batch");
  if (batch * seq * (n_q_heads + n_kv_heads) == 0) return LK_OK;
  LK_REQUIRE(cos && sin && (n_q_heads == 0 || q) && (n_kv_heads == 0 || k), LK_INVALID_ARGUMENT,
             "null pointer");
  cudaStream_t st = as_stream(stream);
  int rc = LK_OK;
  LK_DISPATCH_FLOAT(dtype, T, {
    switch (cos_dtype) {
      case LK_F32: rc = launch_rope<T, float>(q, k, cos, sin, batch, seq, n_q_heads, n_kv_heads, head_dim, cos_batch, backward, st); break;
      case LK_BF16: rc = launch_rope<T, __nv_bfloat16>(q, k, cos, sin, batch, seq, n_q_heads, n_kv_heads, head_dim, cos_batch, backward, st); break;
      case LK_F16: rc = launch_rope<T, __half>(q, k, cos, sin, batch, seq, n_q_heads, n_kv_heads, head_dim, cos_batch, backward, st); break;
      default: return fail(LK_INVALID_ARGUMENT, "unknown cos dtype");
    }
  });
  return rc;
}
