// Persistent, warp-specialised tcgen05 GEMM for sm_100a with the FLCE epilogues.
//
// Tile 128 x 256 x 64 (bf16/fp16 in, fp32 accumulate in TMEM), cta_group::1.
//   warp 0      : TMA producer (one elected lane), 4-stage smem ring, mbarrier full/empty
//   warp 1      : MMA issuer (one lane): 4 x tcgen05.mma (K=16) per stage, commit -> empty
//   warp 2      : TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warps 4..7  : epilogue, one TMEM lane quadrant each -> one output row per thread
// Tiles come from a global atomic counter (dynamic persistent scheduling) and
// are handed to the MMA and epilogue warps through a small smem ring, so the
// TMEM double buffer overlaps tile i's epilogue with tile i+1's MMAs.
//
// Up to two GEMM "problems" share one launch: the FLCE backward runs the dX
// GEMM (long K = V, few tiles) and the dW GEMM (short K = chunk rows, many
// tiles) together, heavy tiles first, so the tail of one fills the other.
//
// Operand layouts (smem, SWIZZLE_128B, UMMA canonical forms; see cute
// mma_sm100_desc.hpp):
//   K-major  : TMA box {64 (K), rows}      -> 8-row groups of 1024 B, SBO = 1024
//   MN-major : TMA boxes {64 (MN), 64 (K)} -> one 8 KB box per 64-wide MN atom,
//              LBO = 8192 (MN atom stride), SBO = 1024 (8-row K group stride)
#pragma once
#include <type_traits>
#include <cuda.h>
#include "gemm_common.cuh"

namespace lk {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, SCHED = 4;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_THREADS = 256;
constexpr int TMEM_COLS = 512;
// stage ring | epilogue staging (4 warps x 2 x 4 KB) | barriers + sched ring + tmem slot
constexpr int AUX_BYTES = 1024;
constexpr int EPI_STAGING_BYTES = 4 * 2 * 4096;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_STAGING_BYTES + AUX_BYTES + 1024;  // + alignment slack

struct Problem {
  int64_t M, N, K;
  int tiles_m, tiles_n, k_blocks;
  // operand load mode: 0 = K-major (one 2D box), 1 = MN-major via one 3D box
  // {64, 64 K, atoms}, 2 = MN-major via one 2D box per 64-wide atom; 3 / 4 / 5 = the same
  // three with a trailing piece coordinate (3D / 4D / 3D maps over [piece][rows][cols])
  int a_mode, b_mode;
  int n_fast;           // tile id -> (m, n): 1 = n varies fastest
  int tma_out;          // 1: epilogue writes through smem staging + TMA store (map mc<p>)
  // Segmented accumulation (fp32 TMA output only): the K loop restarts the TMEM accumulator
  // every seg_kb k-blocks, alternating the two TMEM buffers like separate tiles, and the
  // epilogue stores the first segment and TMA-reduce-adds (fp32, round-to-nearest, in L2) the
  // later ones, each after the previous segment's bulk ops of the same rows have completed
  // (same issuing lane, in order: deterministic).  The tensor core's own fp32 accumulation
  // truncates at every MMA (scripts/probe_tc_accum.py: the error grows with the number of
  // K=16 steps), so long-K fp32 problems keep each truncated run short.  0 = off.
  int seg_kb;
  // Piece-addressed K (fp32 split operands, a_mode / b_mode 3-5): K is n_terms runs of kb_term
  // k-blocks; run t reads piece pa[t] of A and pb[t] of B at K offset (kb mod kb_term) * 64 of
  // that piece (0 = plain K).
  int kb_term;
  unsigned char pa[8], pb[8];
  EpiArgs epi;
  // Device-side row limit (the kept-row FLCE without a host read; CTA-pair kernel only):
  // m_limit != NULL -> only the first max(*m_limit - m_base, 0) rows of M are computed (M tiles
  // past them are skipped); k_limit != NULL -> the K loop stops after max(*k_limit, 1) - k_base
  // rows (K is the row dimension of the dW GEMM).  Rows past the limit hold zeros in the
  // operands, so a limit only removes work.
  const int64_t* m_limit;
  int64_t m_base;
  const int64_t* k_limit;
  int64_t k_base;
};

struct Args {
  Problem prob[2];
  int n_problems;
  int tiles0;           // tiles of problem 0
  int total_tiles;
  int* counter;         // dynamic scheduler (zero at launch)
  uint32_t idesc[2];    // instruction descriptors per problem
};

#if defined(__CUDA_ARCH__)
// ------------------------------------------------------------------ PTX ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_addr(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_expect_tx_addr(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_2d(uint64_t map, uint32_t bar, uint32_t dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(dst), "l"(map), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_3d(uint64_t map, uint32_t bar, uint32_t dst, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(dst), "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tma_4d(uint64_t map, uint32_t bar, uint32_t dst, int x, int y, int z, int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
      ::"r"(dst), "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}
// Operand load modes 1, 2, 4, 5 land the MN-major canonical layout; 0 and 3 the K-major one.
__device__ __forceinline__ int mode_mn(int mode) { return (mode != 0 && mode != 3) ? 1 : 0; }
// One operand box of a k-block (1-CTA kernel): mode as in Problem::a_mode, `atoms` 64-wide MN
// atoms in the box, k0 the K offset (inside the piece for modes 3-5), pc the piece.
__device__ __forceinline__ void load_operand(uint64_t map, int mode, uint32_t bar, uint32_t dst, int k0, int mn0,
                                             int atoms, int pc) {
  switch (mode) {
    case 0: tma_2d(map, bar, dst, k0, mn0); break;
    case 1: tma_3d(map, bar, dst, 0, k0, mn0 >> 6); break;
    case 2:
      for (int j = 0; j < atoms; ++j) tma_2d(map, bar, dst + j * 8192, mn0 + 64 * j, k0);
      break;
    case 3: tma_3d(map, bar, dst, k0, mn0, pc); break;
    case 4: tma_4d(map, bar, dst, 0, k0, mn0 >> 6, pc); break;
    default:
      for (int j = 0; j < atoms; ++j) tma_3d(map, bar, dst + j * 8192, mn0 + 64 * j, k0, pc);
      break;
  }
}
__device__ __forceinline__ void tma_prefetch_2d(uint64_t map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(uint64_t map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(x), "r"(y),
               "r"(z) : "memory");
}
// L2 prefetch of one operand box (mode as in Problem::a_mode/b_mode; mode 2 prefetches its first atom pair).
__device__ __forceinline__ void prefetch_operand(uint64_t map, int mode, int k0, int mn0) {
  if (mode == 0) tma_prefetch_2d(map, k0, mn0);
  else if (mode == 1) tma_prefetch_3d(map, 0, k0, mn0 >> 6);
  else tma_prefetch_2d(map, mn0, k0);
}
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "elect.sync _|P1, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(pred));
  return pred;
}
__device__ __forceinline__ void umma_commit_addr(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2_2d(uint64_t map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2_3d(uint64_t map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(x), "r"(y),
               "r"(z)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// SWIZZLE_128B shared-memory matrix descriptor (sm100 "version 1").
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

struct TileCoord {
  int p, m_blk, n_blk;
};
__device__ __forceinline__ TileCoord decode_tile(const Args& a, int t) {
  TileCoord c;
  c.p = (t >= a.tiles0) ? 1 : 0;
  int lt = c.p ? t - a.tiles0 : t;
  const Problem& P = a.prob[c.p];
  if (P.n_fast) { c.n_blk = lt % P.tiles_n; c.m_blk = lt / P.tiles_n; }
  else { c.m_blk = lt % P.tiles_m; c.n_blk = lt / P.tiles_m; }
  return c;
}

// ------------------------------------------------------------ epilogues ----
template <typename T>
__device__ __forceinline__ void store32(T* dst, const float (&v)[32]) {
  // 32 elements -> 16-byte stores
  constexpr int NV = 16 / sizeof(T);
#pragma unroll
  for (int q = 0; q < 32 / NV; ++q) {
    uint4 raw;
    T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
    for (int i = 0; i < NV; ++i) e[i] = from_f<T>(v[q * NV + i]);
    reinterpret_cast<uint4*>(dst)[q] = raw;
  }
}

// OutT = the chunk buffer's type: T (16-bit logits) or float (fp32 FLCE on split operands,
// where the partials come from the unrounded fp32 logits).
template <typename T, typename OutT = T>
__device__ __forceinline__ void epi_logits(const EpiArgs& e, int64_t grow, int64_t n0, int n_blk,
                                           uint32_t taddr) {
  const bool row_ok = grow < e.M;
  int64_t tcol = -1;
  if (row_ok) {
    int64_t y = e.target[grow];
    if (y != e.ignore_index) tcol = y - e.col_offset;
  }
  const bool cap = e.softcap > 0.f;
  const float inv_cap = cap ? 1.f / e.softcap : 0.f;
  float m = -INFINITY, s = 0.f, sz = 0.f, tv = 0.f;
  bool have_t = false;
  float best_v = -INFINITY;
  int best_i = 0;
  OutT* orow = static_cast<OutT*>(e.out) + grow * e.ldo;
  const bool vec_ok = (e.ldo % (16 / sizeof(OutT))) == 0;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    tmem_wait_ld();
    if (!row_ok) continue;
    const int64_t col0 = n0 + c * 32;
    const int nvalid = (int)(e.N - col0 < 32 ? e.N - col0 : 32);
    if (nvalid <= 0) continue;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float z = __uint_as_float(r[j]);
      if (e.bias && j < nvalid) z += load_any(e.bias, col0 + j, e.out_dtype);
      if (cap) z = sizeof(OutT) == 4 ? e.softcap * tanhf(z * inv_cap) : e.softcap * tanh_fast(z * inv_cap);
      v[j] = round_to<OutT>(z);
    }
    float cm = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) cm = fmaxf(cm, v[j]);
    if (e.want_argmax && cm > best_v) {
      int jj = 0;
#pragma unroll
      for (int j = 31; j >= 0; --j)
        if (j < nvalid && v[j] == cm) jj = j;
      best_v = cm;
      best_i = (int)(col0 + jj);
    }
    const float mn = fmaxf(m, cm);
    float acc = 0.f, zs = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) { acc += __expf(v[j] - mn); zs += v[j]; }
    s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + acc;
    m = mn;
    sz += zs;
    if (tcol >= col0 && tcol < col0 + nvalid) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j == tcol) tv = v[j];
      have_t = true;
    }
    if (nvalid == 32 && vec_ok) {
      store32<OutT>(orow + col0, v);
    } else {
      for (int j = 0; j < nvalid; ++j) orow[col0 + j] = from_f<OutT>(v[j]);
    }
  }
  if (row_ok) {
    e.partials[grow * e.n_parts + n_blk] = make_float4(m, s, sz, e.want_argmax ? __int_as_float(best_i) : 0.f);
    if (have_t) e.tgt_logit[grow] = tv;
  }
}

template <typename T>
__device__ __forceinline__ void epi_store(const EpiArgs& e, int64_t grow, int64_t n0, uint32_t taddr) {
  const bool row_ok = grow < e.M;
  T* orow = static_cast<T*>(e.out) + grow * e.ldo;
  const bool vec_ok = (e.ldo % (16 / sizeof(T))) == 0;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    tmem_wait_ld();
    if (!row_ok) continue;
    const int64_t col0 = n0 + c * 32;
    const int nvalid = (int)(e.N - col0 < 32 ? e.N - col0 : 32);
    if (nvalid <= 0) continue;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = e.alpha * __uint_as_float(r[j]);
    if (nvalid == 32 && vec_ok) store32<T>(orow + col0, v);
    else for (int j = 0; j < nvalid; ++j) orow[col0 + j] = from_f<T>(v[j]);
  }
}

template <typename T>
__device__ __forceinline__ void epi_accum(const EpiArgs& e, int64_t grow, int64_t n0, uint32_t taddr) {
  const bool row_ok = grow < e.M;
  if (!e.acc) {  // weight-dtype accumulation directly in `out`: read, add in fp32, round once
    T* orow = static_cast<T*>(e.out) + grow * e.ldo;
    const bool vec16 = (e.ldo % 8) == 0 && (reinterpret_cast<uintptr_t>(e.out) % 16) == 0;
    uint4 nxt[4];  // the next 32 columns of this row, loaded while TMEM drains the current ones
    auto fetch = [&](int c, uint4 (&dst)[4]) {
      const int64_t col0 = n0 + c * 32;
      if (row_ok && e.beta && vec16 && col0 + 32 <= e.N) {
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = reinterpret_cast<const uint4*>(orow + col0)[q];
      }
    };
    fetch(0, nxt);
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint4 cur[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
      uint32_t r[32];
      tmem_ld32(taddr + c * 32, r);
      if (c + 1 < BN / 32) fetch(c + 1, nxt);
      tmem_wait_ld();
      if (!row_ok) continue;
      const int64_t col0 = n0 + c * 32;
      if (vec16 && col0 + 32 <= e.N) {
        const T* old = reinterpret_cast<const T*>(cur);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (e.beta ? to_f<T>(old[j]) : 0.f) + e.alpha * __uint_as_float(r[j]);
        store32<T>(orow + col0, v);
        continue;
      }
      for (int j = 0; j < 32 && col0 + j < e.N; ++j) {
        const float a = e.beta ? to_f<T>(orow[col0 + j]) : 0.f;
        orow[col0 + j] = from_f<T>(a + e.alpha * __uint_as_float(r[j]));
      }
    }
    return;
  }
  float* arow = e.acc + grow * e.ldacc;
  T* orow = static_cast<T*>(e.out) + grow * e.ldo;
  const bool vec_ok = (e.ldacc % 4) == 0 && (!e.final_out || (e.ldo % 8) == 0);
  float4 nxt[8];
  auto fetch = [&](int c, float4 (&dst)[8]) {
    const int64_t col0 = n0 + c * 32;
    if (row_ok && e.beta && vec_ok && col0 + 32 <= e.N) {
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[q] = reinterpret_cast<const float4*>(arow + col0)[q];
    }
  };
  fetch(0, nxt);
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    float4 cur[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    if (c + 1 < BN / 32) fetch(c + 1, nxt);
    tmem_wait_ld();
    if (!row_ok) continue;
    const int64_t col0 = n0 + c * 32;
    const int nvalid = (int)(e.N - col0 < 32 ? e.N - col0 : 32);
    if (nvalid <= 0) continue;
    float v[32];
    if (nvalid == 32 && vec_ok) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 a = e.beta ? cur[q] : make_float4(0.f, 0.f, 0.f, 0.f);
        v[4 * q + 0] = a.x + __uint_as_float(r[4 * q + 0]);
        v[4 * q + 1] = a.y + __uint_as_float(r[4 * q + 1]);
        v[4 * q + 2] = a.z + __uint_as_float(r[4 * q + 2]);
        v[4 * q + 3] = a.w + __uint_as_float(r[4 * q + 3]);
      }
      if (e.final_out) {
        store32<T>(orow + col0, v);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          reinterpret_cast<float4*>(arow + col0)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    } else {
      for (int j = 0; j < nvalid; ++j) {
        float a = (e.beta ? arow[col0 + j] : 0.f) + __uint_as_float(r[j]);
        if (e.final_out) orow[col0 + j] = from_f<T>(a);
        else arow[col0 + j] = a;
      }
    }
  }
}

template <typename T>
__device__ __forceinline__ void epi_f32(const EpiArgs& e, int64_t grow, int64_t n0, uint32_t taddr) {
  const bool row_ok = grow < e.M;
  float* orow = static_cast<float*>(e.out) + grow * e.ldo;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    tmem_wait_ld();
    if (!row_ok) continue;
    const int64_t col0 = n0 + c * 32;
    for (int j = 0; j < 32; ++j)
      if (col0 + j < e.N) orow[col0 + j] = __uint_as_float(r[j]);
  }
}

// ------------------------------------------- TMA-store epilogues (default) ----
// Each epilogue warp owns 32 rows of the tile and a double-buffered 4 KB staging
// area in shared memory.  A 128-byte row segment (32 fp32 or 64 bf16) per thread
// is written with SWIZZLE_128B placement (16-B chunk j of row r at chunk j ^ (r & 7),
// bank-conflict-free), then one lane issues a TMA bulk tensor store -- or, for the
// fp32 dW accumulator, a TMA reduce-add (the add happens in L2) -- of the 32-row box.
// Out-of-range rows/columns are clipped by the tensor map bounds.  Versus one-row-
// per-thread global stores this turns 32 scattered 16-B accesses per instruction
// into one bulk copy, which frees the L1/shared-memory pipe the mainloop needs.
constexpr int STG_BYTES = 4096;

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tma_store_2d(uint64_t map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
               ::"l"(map), "r"(src), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(uint64_t map, uint32_t src, int x, int y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];"
               ::"l"(map), "r"(src), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

struct Stager {
  uint32_t base;  // this warp's two 4 KB buffers
  int b;
  __device__ __forceinline__ uint32_t acquire(int lane) {
    if (lane == 0) bulk_wait_read1();  // the store that last read this buffer has finished reading
    __syncwarp();
    const uint32_t buf = base + b * STG_BYTES;
    b ^= 1;
    return buf;
  }
  __device__ __forceinline__ void flush(uint64_t map, uint32_t buf, int x, int y, bool reduce, int lane) {
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (reduce) tma_reduce_add_2d(map, buf, x, y);
      else tma_store_2d(map, buf, x, y);
      bulk_commit();
    }
  }
};

// One thread's 128-byte row: eight 16-byte chunks, swizzled.
__device__ __forceinline__ void stage_row(uint32_t buf, int lane, const uint32_t (&w)[32]) {
  const uint32_t row = buf + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    st_shared_v4(row + ((j ^ (lane & 7)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b) {  // one F2FP.PACK_AB, not two F2F
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int N>
__device__ __forceinline__ float tree_max(const float* v) {
  float t[N / 2];
#pragma unroll
  for (int i = 0; i < N / 2; ++i) t[i] = fmaxf(v[2 * i], v[2 * i + 1]);
#pragma unroll
  for (int w = N / 4; w >= 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) t[i] = fmaxf(t[2 * i], t[2 * i + 1]);
  return t[0];
}

// Packed 16-bit pairs for the logits epilogue: one F2FP rounds two logits, the max runs on
// the packed values (HMNMX2 is exact), and the statistics unpack exactly with integer ops --
// no per-element F2F round trip (which sits on the 16/clk conversion pipe).
template <typename T> struct P16;
template <> struct P16<__nv_bfloat16> {
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ float2 unpack(uint32_t u) {
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
  }
  static __device__ __forceinline__ uint32_t hmax(uint32_t a, uint32_t b) {
    __nv_bfloat162 r = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
};
template <> struct P16<__half> {
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ float2 unpack(uint32_t u) { return __half22float2(*reinterpret_cast<__half2*>(&u)); }
  static __device__ __forceinline__ uint32_t hmax(uint32_t a, uint32_t b) {
    __half2 r = __hmax2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
};

// Logit transform of one 64-column group: (+bias) -> (softcap); the caller rounds to the
// logits dtype when it packs.  The branches are warp-uniform and sit outside the unrolled
// element loop.
template <typename T>
__device__ __forceinline__ void logits_values(const EpiArgs& e, const uint32_t (&r0)[32], const uint32_t (&r1)[32],
                                              int64_t col0, int nvalid, float (&v)[64]) {
#pragma unroll
  for (int j = 0; j < 64; ++j) v[j] = __uint_as_float(j < 32 ? r0[j] : r1[j - 32]);
  if (e.bias) {
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (j < nvalid) v[j] += load_any(e.bias, col0 + j, e.out_dtype);
  }
  if (e.softcap > 0.f) {
    const float c = e.softcap, ic = 1.f / e.softcap;
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = c * tanh_fast(v[j] * ic);
  }
}

// 16-bit output (logits with online-softmax partials, or alpha * acc), 64-column groups.
// The statistics use the rounded values, so the finalize's softmax is self-consistent;
// the target logit is not captured here (the finalize reads it from the chunk buffer).
template <typename T, bool LOGITS>
__device__ __forceinline__ void epi_tma16(const EpiArgs& e, uint64_t omap, Stager& sg, int lane, int64_t grow,
                                          int row0, int64_t n0, int n_blk, uint32_t taddr) {
  constexpr float LOG2E = 1.4426950408889634f;
  const bool row_ok = grow < e.M;
  const bool want_sum = LOGITS && e.want_sum;
  const bool want_arg = LOGITS && e.want_argmax;
  float m = -INFINITY, s = 0.f, sz = 0.f;
  float best_v = -INFINITY;  // argmax (token accuracy / predicted tokens): first column of the max
  int best_i = 0;
#pragma unroll 1
  for (int g = 0; g < BN / 64; ++g) {
    uint32_t r0[32], r1[32];
    tmem_ld32(taddr + g * 64, r0);
    tmem_ld32(taddr + g * 64 + 32, r1);
    tmem_wait_ld();
    const int64_t col0 = n0 + g * 64;
    uint32_t w[32];
    if (LOGITS) {
      using H = P16<T>;
      const int64_t rem = e.N - col0;
      const int nvalid = (int)(rem < 64 ? (rem > 0 ? rem : 0) : 64);
      // 1. (+bias) (softcap) and round to the logits dtype: one F2FP per pair of columns
      if (!e.bias && !(e.softcap > 0.f)) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          w[j] = H::pack(__uint_as_float(r0[2 * j]), __uint_as_float(r0[2 * j + 1]));
          w[16 + j] = H::pack(__uint_as_float(r1[2 * j]), __uint_as_float(r1[2 * j + 1]));
        }
      } else {
        float v[64];
        logits_values<T>(e, r0, r1, col0, nvalid, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) w[j] = H::pack(v[2 * j], v[2 * j + 1]);
      }
      // 2. online-softmax statistics of the ROUNDED values (self-consistent with the finalize)
      if (want_arg && nvalid > 0) {  // warp-uniform option branch, off on the default path
        float gm = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 z = H::unpack(w[j]);
          if (2 * j < nvalid) gm = fmaxf(gm, z.x);
          if (2 * j + 1 < nvalid) gm = fmaxf(gm, z.y);
        }
        if (gm > best_v) {  // strict: an earlier group keeps ties (first index wins)
          int jj = 0;
#pragma unroll
          for (int j = 31; j >= 0; --j) {  // static indices: w stays in registers
            const float2 z = H::unpack(w[j]);
            if (2 * j + 1 < nvalid && z.y == gm) jj = 2 * j + 1;
            if (2 * j < nvalid && z.x == gm) jj = 2 * j;
          }
          best_v = gm;
          best_i = (int)(col0 + jj);
        }
      }
      if (nvalid == 64) {
        uint32_t mx[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) mx[j] = H::hmax(w[2 * j], w[2 * j + 1]);
#pragma unroll
        for (int wd = 8; wd >= 1; wd >>= 1)
#pragma unroll
          for (int j = 0; j < wd; ++j) mx[j] = H::hmax(mx[j], mx[j + wd]);
        const float2 gm2 = H::unpack(mx[0]);
        const float mn = fmaxf(m, fmaxf(gm2.x, gm2.y));
        const float2 l2e2 = make_float2(LOG2E, LOG2E), nml2 = make_float2(-mn * LOG2E, -mn * LOG2E);
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, z0 = a0, z1 = a0;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 za = H::unpack(w[j]), zb = H::unpack(w[j + 1]);
          const float2 ta = __ffma2_rn(za, l2e2, nml2), tb = __ffma2_rn(zb, l2e2, nml2);
          a0 = __fadd2_rn(a0, make_float2(ex2f(ta.x), ex2f(ta.y)));
          a1 = __fadd2_rn(a1, make_float2(ex2f(tb.x), ex2f(tb.y)));
          if (want_sum) { z0 = __fadd2_rn(z0, za); z1 = __fadd2_rn(z1, zb); }
        }
        if (want_sum) sz += (z0.x + z0.y) + (z1.x + z1.y);
        s = s * ex2f((m - mn) * LOG2E) + ((a0.x + a0.y) + (a1.x + a1.y));  // m = -inf first: ex2(-inf) = 0
        m = mn;
      } else if (nvalid > 0) {
        float cm = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 z = H::unpack(w[j]);
          if (2 * j < nvalid) cm = fmaxf(cm, z.x);
          if (2 * j + 1 < nvalid) cm = fmaxf(cm, z.y);
        }
        const float mn = fmaxf(m, cm);
        float a = 0.f, zs = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 z = H::unpack(w[j]);
          if (2 * j < nvalid) { a += ex2f((z.x - mn) * LOG2E); zs += z.x; }
          if (2 * j + 1 < nvalid) { a += ex2f((z.y - mn) * LOG2E); zs += z.y; }
        }
        s = s * ex2f((m - mn) * LOG2E) + a;
        m = mn;
        if (want_sum) sz += zs;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        w[j] = pack2<T>(e.alpha * __uint_as_float(r0[2 * j]), e.alpha * __uint_as_float(r0[2 * j + 1]));
        w[16 + j] = pack2<T>(e.alpha * __uint_as_float(r1[2 * j]), e.alpha * __uint_as_float(r1[2 * j + 1]));
      }
    }
    const uint32_t buf = sg.acquire(lane);
    stage_row(buf, lane, w);
    // EPI_ACCUM into a 16-bit grad_w (weight-dtype accumulation): later chunks reduce-add
    sg.flush(omap, buf, (int)col0, row0, !LOGITS && e.kind == EPI_ACCUM && e.beta != 0, lane);
  }
  if (LOGITS && row_ok)
    e.partials[grow * e.n_parts + n_blk] = make_float4(m, s, sz, want_arg ? __int_as_float(best_i) : 0.f);
}

// fp32 output: plain store (F32 / first dW chunk) or reduce-add (later dW chunks).
__device__ __forceinline__ void epi_tma32(uint64_t omap, Stager& sg, int lane, int row0, int64_t n0, bool reduce,
                                          uint32_t taddr) {
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    tmem_wait_ld();
    const uint32_t buf = sg.acquire(lane);
    stage_row(buf, lane, r);
    sg.flush(omap, buf, (int)(n0 + c * 32), row0, reduce, lane);
  }
}

// Segmented accumulation helpers (Problem::seg_kb).
__device__ __forceinline__ int seg_len(const Problem& P) { return P.seg_kb > 0 ? P.seg_kb : P.k_blocks; }
__device__ __forceinline__ int seg_count(const Problem& P) {
  return P.seg_kb > 0 ? (P.k_blocks + P.seg_kb - 1) / P.seg_kb : 1;
}
// One segment's fp32 partial: the first stores, later ones reduce-add after this lane's
// earlier bulk ops (which cover exactly these rows) have been performed.
__device__ __forceinline__ void epi_segment(uint64_t omap, Stager& sg, int lane, int row0, int64_t n0, int seg,
                                            uint32_t taddr) {
  if (seg > 0 && lane == 0) bulk_wait_all();
  __syncwarp();
  epi_tma32(omap, sg, lane, row0, n0, seg > 0, taddr);
}

// Dispatch one tile's epilogue for this warp.
template <typename T>
__device__ __forceinline__ void run_epilogue(const Problem& P, uint64_t omap, Stager& sg, int lane, int64_t grow,
                                             int row0, int64_t n0, int n_blk, uint32_t taddr) {
  const EpiArgs& e = P.epi;
  if (P.tma_out) {
    switch (e.kind) {
      case EPI_LOGITS: epi_tma16<T, true>(e, omap, sg, lane, grow, row0, n0, n_blk, taddr); break;
      case EPI_STORE: epi_tma16<T, false>(e, omap, sg, lane, grow, row0, n0, n_blk, taddr); break;
      case EPI_ACCUM:
        if (e.acc) epi_tma32(omap, sg, lane, row0, n0, e.beta != 0, taddr);
        else epi_tma16<T, false>(e, omap, sg, lane, grow, row0, n0, n_blk, taddr);
        break;
      default: epi_tma32(omap, sg, lane, row0, n0, false, taddr); break;
    }
    return;
  }
  switch (e.kind) {
    case EPI_LOGITS:
      if (e.out_dtype == LK_F32) epi_logits<T, float>(e, grow, n0, n_blk, taddr);
      else epi_logits<T>(e, grow, n0, n_blk, taddr);
      break;
    case EPI_STORE: epi_store<T>(e, grow, n0, taddr); break;
    case EPI_ACCUM: epi_accum<T>(e, grow, n0, taddr); break;
    default: epi_f32<T>(e, grow, n0, taddr); break;
  }
}
#endif  // __CUDA_ARCH__

// ---------------------------------------------------------------- kernel ----
template <typename T>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap ma0, const __grid_constant__ CUtensorMap mb0,
            const __grid_constant__ CUtensorMap ma1, const __grid_constant__ CUtensorMap mb1,
            const __grid_constant__ CUtensorMap mc0, const __grid_constant__ CUtensorMap mc1,
            const __grid_constant__ Args args) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint8_t* sStg = smem + STAGES * STAGE_BYTES;
  uint64_t* aux = reinterpret_cast<uint64_t*>(sStg + EPI_STAGING_BYTES);
  uint64_t* full = aux;                    // [STAGES]
  uint64_t* empty = full + STAGES;         // [STAGES]
  uint64_t* tfull = empty + STAGES;        // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint64_t* sfull = tempty + 2;            // [SCHED]
  uint64_t* sempty = sfull + SCHED;        // [SCHED]
  int* stile = reinterpret_cast<int*>(sempty + SCHED);  // [SCHED]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stile + SCHED);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    for (int i = 0; i < SCHED; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], 5); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&ma0); tma_prefetch_desc(&mb0);
    if (args.n_problems > 1) { tma_prefetch_desc(&ma1); tma_prefetch_desc(&mb1); }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (warp-converged, one elected issuer) =====================
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB), full0 = smem_u32(full), empty0 = smem_u32(empty);
    for (int it = 0;; ++it) {
      const int slot = it % SCHED;
      int tile = 0;
      if (lane == 0) {
        mbar_wait(&sempty[slot], ((it / SCHED) & 1) ^ 1);
        tile = atomicAdd(args.counter, 1);
        if (tile >= args.total_tiles) tile = -1;
        stile[slot] = tile;
        mbar_arrive(&sfull[slot]);
      }
      tile = __shfl_sync(0xffffffffu, tile, 0);
      if (tile < 0) break;
      const TileCoord tcd = decode_tile(args, tile);
      const int p = tcd.p;
      const int a_mode = p ? args.prob[1].a_mode : args.prob[0].a_mode;
      const int b_mode = p ? args.prob[1].b_mode : args.prob[0].b_mode;
      const int kblocks = p ? args.prob[1].k_blocks : args.prob[0].k_blocks;
      const uint64_t ma = reinterpret_cast<uint64_t>(p ? &ma1 : &ma0);
      const uint64_t mb = reinterpret_cast<uint64_t>(p ? &mb1 : &mb0);
      const int m0 = tcd.m_blk * BM, n0 = tcd.n_blk * BN;
      const int kbt = p ? args.prob[1].kb_term : args.prob[0].kb_term;
      const Problem& PP = args.prob[p];
      int term = 0, kt = 0;  // piece-addressed K (kbt > 0): run index and k-block inside the run
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait_addr(empty0 + stage * 8, phase ^ 1);
        if (elect_one()) {
          const uint32_t fb = full0 + stage * 8;
          mbar_expect_tx_addr(fb, STAGE_BYTES);
          const uint32_t a_dst = sA0 + stage * A_BYTES, b_dst = sB0 + stage * B_BYTES;
          // mode 0: K-major 2D {64 K, rows}; 1: MN-major 3D {64, 64 K, atoms}; 2: MN-major 2D per atom;
          // 3-5: the same with a piece coordinate
          if (kbt == 0) {
            load_operand(ma, a_mode, fb, a_dst, kb * BK, m0, BM / 64, 0);
            load_operand(mb, b_mode, fb, b_dst, kb * BK, n0, BN / 64, 0);
          } else {
            load_operand(ma, a_mode, fb, a_dst, kt * BK, m0, BM / 64, PP.pa[term]);
            load_operand(mb, b_mode, fb, b_dst, kt * BK, n0, BN / 64, PP.pb[term]);
          }
        }
        if (kbt && ++kt == kbt) { kt = 0; ++term; }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (warp-converged, one elected issuer) =====================
    int stage = 0;
    uint32_t phase = 0, use = 0;  // use: accumulations issued so far (TMEM buffer = use & 1)
    const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB), full0 = smem_u32(full), empty0 = smem_u32(empty);
    for (int it = 0;; ++it) {
      const int slot = it % SCHED;
      mbar_wait(&sfull[slot], (it / SCHED) & 1);
      const int tile = stile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[slot]);
      if (tile < 0) break;
      const TileCoord tcd = decode_tile(args, tile);
      const int p = tcd.p;
      const int a_mn = tc::mode_mn(p ? args.prob[1].a_mode : args.prob[0].a_mode);
      const int b_mn = tc::mode_mn(p ? args.prob[1].b_mode : args.prob[0].b_mode);
      const int kblocks = p ? args.prob[1].k_blocks : args.prob[0].k_blocks;
      const int seg_kb = seg_len(args.prob[p]);
      const uint32_t idesc = p ? args.idesc[1] : args.idesc[0];
      // descriptors of stage 0 / k 0; stage and K advances only touch the start-address field
      const uint64_t a_desc0 = make_desc(sA0, a_mn ? 8192u : 16u, 1024u);
      const uint64_t b_desc0 = make_desc(sB0, b_mn ? 8192u : 16u, 1024u);
      const uint32_t a_k16 = a_mn ? (2048u >> 4) : (32u >> 4);   // per UMMA_K=16 step
      const uint32_t b_k16 = b_mn ? (2048u >> 4) : (32u >> 4);
      int buf = 0, ks = 0;
      uint32_t d_tmem = 0;
      for (int kb = 0; kb < kblocks; ++kb) {
        if (ks == 0) {  // a new accumulation (tile, or segment of a segmented tile): next TMEM buffer
          buf = (int)(use & 1);
          mbar_wait(&tempty[buf], ((use >> 1) & 1) ^ 1);
          tc_fence_after();
          d_tmem = tmem_base + buf * BN;
        }
        mbar_wait_addr(full0 + stage * 8, phase);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad = a_desc0 + (uint64_t)((stage * A_BYTES) >> 4);
          const uint64_t bd = b_desc0 + (uint64_t)((stage * B_BYTES) >> 4);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_f16(d_tmem, ad + k * a_k16, bd + k * b_k16, idesc, (ks | k) != 0 ? 1u : 0u);
          umma_commit_addr(empty0 + stage * 8);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        if (++ks == seg_kb || kb == kblocks - 1) {
          if (elect_one()) umma_commit(&tfull[buf]);
          __syncwarp();
          ks = 0;
          ++use;
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp & 3;
    Stager sg{smem_u32(sStg) + (uint32_t)(q * 2 * STG_BYTES), 0};
    uint32_t use = 0;
    for (int it = 0;; ++it) {
      const int slot = it % SCHED;
      mbar_wait(&sfull[slot], (it / SCHED) & 1);
      const int tile = stile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[slot]);
      if (tile < 0) break;
      const TileCoord tcd = decode_tile(args, tile);
      const Problem& P = args.prob[tcd.p];
      const uint64_t omap = reinterpret_cast<uint64_t>(tcd.p ? &mc1 : &mc0);
      const int row0 = tcd.m_blk * BM + q * 32;
      const int64_t grow = (int64_t)row0 + lane;
      const int64_t n0 = (int64_t)tcd.n_blk * BN;
      const int nseg = seg_count(P);
      for (int sgi = 0; sgi < nseg; ++sgi, ++use) {
        const int buf = (int)(use & 1);
        mbar_wait(&tfull[buf], (use >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + buf * BN + ((uint32_t)(q * 32) << 16);
        if (nseg > 1) epi_segment(omap, sg, lane, row0, n0, sgi, taddr);
        else run_epilogue<T>(P, omap, sg, lane, grow, row0, n0, tcd.n_blk, taddr);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
#endif
}

// ------------------------------------------------------------------ host ----
// Instruction descriptor for kind::f16 (cute UMMA::InstrDescriptor bit layout):
// c_format F32 @4, a/b format @7/@10 (0 = F16, 1 = BF16), a/b major @15/@16,
// N>>3 @17, M>>4 @24.
inline uint32_t make_idesc(int dtype, int a_mn, int b_mn) {
  uint32_t fmt = dtype == LK_BF16 ? 1u : 0u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// One GEMM operand as the TMA sees it: a row-major [outer, inner] matrix.
struct TmaOperand {
  const void* ptr;
  int64_t inner, outer;  // elements
  int64_t row_elems;     // row stride in elements
  int mn_major;          // 0: inner dim is K; 1: inner dim is M/N
  int pieces = 0;        // > 0: `pieces` such matrices, piece_elems apart (load modes 3-5)
  int64_t piece_elems = 0;
};

// Encodes the operand's tensor map and returns its load mode (0/1/2, see Problem).
int encode_operand(CUtensorMap* map, const TmaOperand& op, int dtype, int rows_in_box, int* mode);
bool tma_ok(const TmaOperand& op);

// Launch one or two problems in a single persistent launch.
// Problem p: C[M, N] = A·B with A given by `a[p]` and B by `b[p]`.
// cta_group: 1 = single-CTA 128x256 tiles, 2 = CTA-pair 256x256 tiles, 0 = default (pair).
// register_epilogue: force the register-path epilogue (test hook for the 16-bit read-add path)
int launch_tc_gemm(const TmaOperand* a, const TmaOperand* b, Problem* probs, int n_problems, int dtype,
                   int* counter, cudaStream_t st, int cta_group = 0, bool register_epilogue = false);

}  // namespace tc
}  // namespace lk
