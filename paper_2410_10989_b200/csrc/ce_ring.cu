// Standalone cross entropy: persistent TMA-ring row streaming (default path).
//
// The reference streams each row twice -- statistics, then the in-place gradient
// rewrite (rowfuse/ops.py:530-551; Liger LK/ops/cross_entropy.py:118-246).  Here one
// CTA per SM walks its rows (b, b + G, ...) as a sequence of 16 KB pieces: a producer
// warp pulls pass-1 pieces, then pass-2 pieces of the same row, into a ring of S
// shared-memory stages with 1D bulk copies, and keeps loading the next row while the
// consumers finish the current one.  The pass-2 copy of a piece was read from HBM a
// few hundred KB earlier (148 rows x 250 KB in flight << 126 MB L2), so HBM sees one
// read and one write per logit.
//
// Per logit the kernel issues ~10 instructions (packed fp32x2 FFMA2/FADD2, one MUFU
// ex2 per pass) across 16 consumer warps: at 8192 x 128256 that is close to both the
// HBM time and the MUFU time (2 ex2 per logit at 16/clk/SM), so option handling is
// compile-time (softcap, label smoothing) and the ragged-piece masking and the target
// correction are hoisted out of the per-element path.
//
// Consumer warp c owns 16-byte vectors [c*64, (c+1)*64) of every piece, keeps a running
// online-softmax (max, sumexp, sum) per lane, and the warps combine per row through
// shared memory in warp order (deterministic).  Every warp consumes every piece in
// sequence order, so each fill of a stage is waited for by a warp that consumed the
// previous fill of that stage: mbarrier parities cannot alias.
#include "ce.cuh"
#include "ring.cuh"

namespace lk {
namespace cer {

constexpr int NC = 16;
constexpr int THREADS = (NC + 1) * 32;
constexpr uint32_t PIECE = 32768;             // bytes per ring stage
constexpr int VPW = PIECE / 16 / NC;          // 16-byte vectors per warp per piece (128)
constexpr int KPL = VPW / 32;                 // per lane (4)
constexpr float L2E = 1.4426950408889634f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 ex2(float2 x) { return make_float2(ex2(x.x), ex2(x.y)); }

using ring::Pairs;

struct Smem {
  float4 red[2][NC];
  float wz[2][NC];   // class weights + smoothing, FLCE finalize: per-warp sum_c w_c z_c after pass 2
  float2 am[2][NC];  // per-warp argmax (value, index bits) for token accuracy / predicted tokens
  float zt[2];
};

template <typename T, bool CAP>
__device__ __forceinline__ float2 capped(float2 z, float cap, float inv_cap) {
  if constexpr (!CAP) {
    return z;
  } else {
    constexpr bool ACC = sizeof(T) == 4;
    const float2 u = __fmul2_rn(z, make_float2(inv_cap, inv_cap));
    const float2 t = ACC ? make_float2(tanhf(u.x), tanhf(u.y)) : make_float2(tanh_fast(u.x), tanh_fast(u.y));
    return __fmul2_rn(t, make_float2(cap, cap));
  }
}

// PART: FLCE finalize -- the logits GEMM epilogue already wrote per-(row, 256-column tile)
// (max, sumexp, sum) partials and the softcapped, rounded logits, so the statistics pass is a
// combine of ~V/256 partials and only the gradient pass streams the row (one read + one
// write per logit, rowfuse/flce.py:155-157).
// W: class weights together with label smoothing (compile-time, so the common variants carry
// no per-element weight branch).
template <typename T, bool CAP, bool LS, bool PART, bool W>
__global__ void __launch_bounds__(THREADS, 1) ce_ring_kernel(CeRowArgs a, int stages) {
  using P = Pairs<T>;
  constexpr int NP = P::NP;
  constexpr int NV = 16 / sizeof(T);
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * PIECE);
  uint64_t* empty = full + stages;
  Smem* sh = reinterpret_cast<Smem*>(empty + stages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t rows = a.rows, n = a.n_cols;
  const int64_t n_local = rows > b ? (rows - b + G - 1) / G : 0;
  const int64_t row_bytes = n * (int64_t)sizeof(T);
  const int64_t npc = (row_bytes + PIECE - 1) / PIECE;
  const int passes = PART ? (a.compute_grad ? 1 : 0) : (a.compute_grad ? 2 : 1);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { ring::mbar_init(&full[s], 1); ring::mbar_init(&empty[s], NC); }
    ring::fence_init();
  }
  __syncthreads();

  if (warp == NC) {  // producer
    if (lane == 0) {
      ring::Cursor cur(stages);
      for (int64_t i = 0; i < n_local; ++i) {
        const int64_t row = b + i * G;
        if (a.target[row] == a.ignore_index) continue;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.x) + row * a.ld * (int64_t)sizeof(T);
        for (int p = 0; p < passes; ++p)
          for (int64_t j = 0; j < npc; ++j, cur.next()) {
            const int s = cur.s;
            if (cur.wrapped) ring::wait(&empty[s], cur.phase ^ 1u);
            const uint32_t bytes = (uint32_t)min((int64_t)PIECE, row_bytes - j * PIECE);
            ring::expect_tx(&full[s], bytes);
            ring::bulk_g2s(sm + (size_t)s * PIECE, src + j * PIECE, bytes, &full[s]);
          }
      }
    }
    return;
  }

  const float cap = a.softcap, inv_cap = CAP ? 1.f / a.softcap : 0.f;
  const int tid = threadIdx.x;
  const float2 l2e2 = make_float2(L2E, L2E);
  const bool want_arg = a.correct_rows || a.pred_rows;
  ring::Cursor cur(stages);
  int par = 0;
  // per-piece bookkeeping in 32-bit shared-window addresses and int column offsets
  const uint32_t sbase = ring::s_u32(sm) + (uint32_t)(warp * VPW + lane) * 16u;
  const uint32_t full_a = ring::s_u32(full), empty_a = ring::s_u32(empty);
  const int npc32 = (int)npc;
  const int tail_nvec = (int)((row_bytes - (npc - 1) * (int64_t)PIECE) / 16);
  const int v0 = warp * VPW + lane;
  int64_t zero_end = INT64_MAX;  // local rows at or past it: ignored-row zero writes skipped
  if (a.zero_limit) {
    const int64_t lim = *a.zero_limit < 1 ? 1 : *a.zero_limit;
    zero_end = (lim + 255) / 256 * 256 - a.zero_base;
  }
  // class weights with label smoothing: the smoothing sum is sum_c w_c z_c and the gradient
  // gains -eps w_c per column (weights by global column; runtime-uniform branch)
  const float* wcol = W ? a.class_weight + a.col_offset : nullptr;
  for (int64_t i = 0; i < n_local; ++i) {
    const int64_t row = b + i * G;
    T* xr = static_cast<T*>(a.x) + row * a.ld;
    const int64_t y = a.target[row];
    if (y == a.ignore_index) {
      if (a.compute_grad && row < zero_end)
        for (int64_t v = tid; v < n / NV; v += NC * 32) ring::stg128(xr + v * NV, make_uint4(0, 0, 0, 0));
      if (tid == 0) {
        if (a.loss_rows) a.loss_rows[row] = 0.f;
        if (a.z_loss_rows) a.z_loss_rows[row] = 0.f;
        if (a.correct_rows) a.correct_rows[row] = 0.f;
        if (a.pred_rows) a.pred_rows[row] = -1;
      }
      continue;
    }
    const int64_t yl = y - a.col_offset;
    if (tid == 0) {
      float zt = 0.f;
      if (PART && a.row_stats) {
        zt = a.row_stats[row].w;  // global target logit (the target may live on another shard)
      } else if (yl >= 0 && yl < n) {
        zt = to_f<T>(xr[yl]);  // read before any pass-2 write of this row (after the barrier below)
        if (CAP && !PART) zt = cap * tanhf(zt * inv_cap);
      }
      sh->zt[par] = zt;
    }
    // ---- pass 1: online (max, sumexp[, sum]) ----
    float m = -INFINITY, se = 0.f;
    float2 sz2 = make_float2(0.f, 0.f);
    float av = -INFINITY;  // argmax (option): value, first column
    int ai = 0x7fffffff;
    if constexpr (PART) {
      if (a.row_stats) {  // vocab-parallel: the all-reduced global row statistics
        if (tid == 0) {
          const float4 st = a.row_stats[row];
          m = st.x; se = st.y; sz2.x = st.z;
        }
      } else {
        const float4* pp = a.partials + row * a.n_parts;
        for (int64_t jp = tid; jp < a.n_parts; jp += NC * 32) {
          const float4 q = pp[jp];
          ms_combine(m, se, q.x, q.y);
          sz2.x += q.z;
          if (want_arg) am_merge(av, ai, q.x, __float_as_int(q.w));
        }
      }
    }
    for (int j = 0; j < (PART ? 0 : npc32); ++j, cur.next()) {
      const int s = cur.s;
      ring::wait(full_a + 8u * (uint32_t)s, cur.phase);
      const int nvec = j == npc32 - 1 ? tail_nvec : (int)(PIECE / 16);
      const uint32_t st = sbase + (uint32_t)s * PIECE;
      uint4 raw[KPL];
#pragma unroll
      for (int k = 0; k < KPL; ++k) raw[k] = v0 + 32 * k < nvec ? ring::lds128(st + 512u * k) : make_uint4(0, 0, 0, 0);
      ring::release_after_loads(empty_a + 8u * (uint32_t)s, raw, lane);
      float2 z[KPL][NP];
      float lmax = -INFINITY;
      if (nvec == (int)(PIECE / 16)) {  // whole piece (all but a ragged row tail): no masking
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
          P::unpack(raw[k], z[k]);
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            z[k][e] = capped<T, CAP>(z[k][e], cap, inv_cap);
            lmax = fmaxf(lmax, fmaxf(z[k][e].x, z[k][e].y));
          }
        }
        const float mn = fmaxf(m, lmax);
        const float2 nmb = make_float2(-mn * L2E, -mn * L2E);
        float2 acc = make_float2(0.f, 0.f);
        const float* wp = W ? wcol + (int64_t)j * (PIECE / sizeof(T)) + v0 * NV : nullptr;
#pragma unroll
        for (int k = 0; k < KPL; ++k)
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            acc = __fadd2_rn(acc, ex2(__ffma2_rn(z[k][e], l2e2, nmb)));
            if constexpr (W) sz2 = __ffma2_rn(z[k][e], __ldg(reinterpret_cast<const float2*>(wp + 32 * k * NV + 2 * e)), sz2);
            else if (LS) sz2 = __fadd2_rn(sz2, z[k][e]);
          }
        se = se * ex2((m - mn) * L2E) + (acc.x + acc.y);  // m = -inf: ex2(-inf) = 0, se = 0
        m = mn;
        if (want_arg && lmax > av) {  // option; strict: earlier columns keep ties
          const int cbase = j * (int)(PIECE / sizeof(T));
#pragma unroll
          for (int k = KPL - 1; k >= 0; --k)
#pragma unroll
            for (int e = NP - 1; e >= 0; --e) {
              const int c = cbase + (v0 + 32 * k) * NV + 2 * e;
              if (z[k][e].y == lmax) ai = c + 1;
              if (z[k][e].x == lmax) ai = c;
            }
          av = lmax;
        }
      } else {
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
          P::unpack(raw[k], z[k]);
          const bool ok = v0 + 32 * k < nvec;
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            z[k][e] = ok ? capped<T, CAP>(z[k][e], cap, inv_cap) : make_float2(-INFINITY, -INFINITY);
            lmax = fmaxf(lmax, fmaxf(z[k][e].x, z[k][e].y));
          }
        }
        if (lmax == -INFINITY) continue;  // lane holds no logit of this piece
        const float mn = fmaxf(m, lmax);
        const float2 nmb = make_float2(-mn * L2E, -mn * L2E);
        float2 acc = make_float2(0.f, 0.f);
        const float* wp = W ? wcol + (int64_t)j * (PIECE / sizeof(T)) + v0 * NV : nullptr;
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
          if (v0 + 32 * k >= nvec) continue;
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            acc = __fadd2_rn(acc, ex2(__ffma2_rn(z[k][e], l2e2, nmb)));
            if constexpr (W) sz2 = __ffma2_rn(z[k][e], __ldg(reinterpret_cast<const float2*>(wp + 32 * k * NV + 2 * e)), sz2);
            else if (LS) sz2 = __fadd2_rn(sz2, z[k][e]);
          }
        }
        se = (m == -INFINITY ? 0.f : se * ex2((m - mn) * L2E)) + (acc.x + acc.y);
        m = mn;
        if (want_arg && lmax > av) {
          const int cbase = j * (int)(PIECE / sizeof(T));
#pragma unroll
          for (int k = KPL - 1; k >= 0; --k)
#pragma unroll
            for (int e = NP - 1; e >= 0; --e) {
              const int c = cbase + (v0 + 32 * k) * NV + 2 * e;
              if (z[k][e].y == lmax) ai = c + 1;
              if (z[k][e].x == lmax) ai = c;
            }
          av = lmax;
        }
      }
    }
    float sz = sz2.x + sz2.y;
    warp_ms(m, se);
    if (LS) sz = warp_sum(sz);
    if (want_arg) warp_am(av, ai);
    if (lane == 0) {
      sh->red[par][warp] = make_float4(m, se, sz, 0.f);
      sh->am[par][warp] = make_float2(av, __int_as_float(ai));
    }
    ring::consumers_sync(1, NC * 32);
    m = -INFINITY; se = 0.f; sz = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {  // fixed warp order: deterministic
      const float4 r = sh->red[par][c];
      ms_combine(m, se, r.x, r.y);
      sz += r.z;
    }
    const float zy = sh->zt[par];
    if (want_arg && tid == 0) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int c = 0; c < NC; ++c) am_merge(bv, bi, sh->am[par][c].x, __float_as_int(sh->am[par][c].y));
      const int64_t am = (int64_t)bi + a.col_offset;
      if (a.pred_rows) a.pred_rows[row] = am;
      if (a.correct_rows) a.correct_rows[row] = am == y ? 1.f : 0.f;
    }
    par ^= 1;
    const float lse = m + logf(se);
    // reduction (MEAN), token scaling and class weights folded into per-row coefficients
    const RowCoef rcf = ce_row_coefs<T>(a, lse, zy, sz, y);
    // FLCE finalize with class weights + smoothing: the epilogue partials carry the unweighted
    // sum, so sum_c w_c z_c is accumulated in pass 2 and the loss written after it
    constexpr bool late_loss = PART && W;
    if (tid == 0 && !late_loss) {  // LK/ops/cross_entropy.py:259-289
      if (a.loss_rows) a.loss_rows[row] = rcf.loss;
      if (a.z_loss_rows) a.z_loss_rows[row] = rcf.zl;
    }
    if (!a.compute_grad) continue;
    // ---- pass 2: gradient in place (LK/ops/cross_entropy.py:181-246) ----
    const float coef = rcf.pc / se;
    const float2 nmb = make_float2(-m * L2E, -m * L2E);
    const float2 coef2 = make_float2(coef, coef);
    const float2 neps2 = make_float2(rcf.ceps, rcf.ceps);
    const float hit_s = rcf.chit;
    float2 wz2 = make_float2(0.f, 0.f);  // late_loss: sum_c w_c z_c
    for (int j = 0; j < npc32; ++j, cur.next()) {
      const int s = cur.s;
      ring::wait(full_a + 8u * (uint32_t)s, cur.phase);
      const int nvec = j == npc32 - 1 ? tail_nvec : (int)(PIECE / 16);
      const uint32_t st = sbase + (uint32_t)s * PIECE;
      uint4 raw[KPL];
#pragma unroll
      for (int k = 0; k < KPL; ++k) raw[k] = v0 + 32 * k < nvec ? ring::lds128(st + 512u * k) : make_uint4(0, 0, 0, 0);
      ring::release_after_loads(empty_a + 8u * (uint32_t)s, raw, lane);
      const int64_t col0 = (int64_t)j * (PIECE / sizeof(T));
      T* xp = xr + col0 + (int64_t)v0 * NV;  // this lane's first vector of the piece
      const float* wp = W ? wcol + col0 + (int64_t)v0 * NV : nullptr;
      // target column relative to that vector, as a 32-bit value (far away when not in the piece)
      const int64_t trel64 = yl - col0 - (int64_t)v0 * NV;
      const int trel = trel64 >= -(int64_t)(PIECE / sizeof(T)) && trel64 < (int64_t)(PIECE / sizeof(T)) ? (int)trel64 : INT_MIN / 2;
#pragma unroll
      for (int k = 0; k < KPL; ++k) {
        const int v = v0 + 32 * k;
        if (v < nvec) {
          float2 z[NP];
          P::unpack(raw[k], z);
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            float2 zz = z[e], dc = make_float2(1.f, 1.f);
            if (CAP) {
              const float2 u = __fmul2_rn(zz, make_float2(inv_cap, inv_cap));
              float2 t = u;  // PART: the buffer already holds cap * tanh(z / cap)
              if (!PART) {
                t = sizeof(T) == 4 ? make_float2(tanhf(u.x), tanhf(u.y)) : make_float2(tanh_fast(u.x), tanh_fast(u.y));
                zz = __fmul2_rn(t, make_float2(cap, cap));
              }
              dc = __ffma2_rn(__fmul2_rn(t, t), make_float2(-1.f, -1.f), make_float2(1.f, 1.f));  // 1 - t^2
            }
            float2 g;
            if constexpr (W) {
              const float2 wv = __ldg(reinterpret_cast<const float2*>(wp + 32 * k * NV + 2 * e));
              g = __ffma2_rn(ex2(__ffma2_rn(zz, l2e2, nmb)), coef2, __fmul2_rn(neps2, wv));
              if (late_loss) wz2 = __ffma2_rn(zz, wv, wz2);
            } else {
              g = __ffma2_rn(ex2(__ffma2_rn(zz, l2e2, nmb)), coef2, neps2);
            }
            if (CAP) g = __fmul2_rn(g, dc);
            z[e] = g;
          }
          ring::stg128(xp + 32 * k * NV, P::pack(z));
          // the target column: rewrite that one element after the vector store (same thread,
          // program order) -- keeps the per-element path free of the compare
          const uint32_t off = (uint32_t)(trel - 32 * k * NV);
          if (off < (uint32_t)NV) {
            const uint32_t word = off * sizeof(T) / 4;
            const uint32_t u = word == 0 ? raw[k].x : word == 1 ? raw[k].y : word == 2 ? raw[k].z : raw[k].w;
            float zt;
            if constexpr (sizeof(T) == 4) zt = __uint_as_float(u);
            else {
              const uint16_t hbits = (off & 1) ? (uint16_t)(u >> 16) : (uint16_t)(u & 0xffffu);
              zt = to_f<T>(*reinterpret_cast<const T*>(&hbits));
            }
            float dct = 1.f;
            if (CAP) {
              float t = zt * inv_cap;
              if (!PART) {
                t = sizeof(T) == 4 ? tanhf(t) : tanh_fast(t);
                zt = cap * t;
              }
              dct = 1.f - t * t;
            }
            const float ce = W ? neps2.x * wcol[yl] : neps2.x;
            const float gt = (ex2(fmaf(zt, L2E, nmb.x)) * coef + ce - hit_s) * dct;
            xr[yl] = from_f<T>(gt);
          }
        }
      }
    }
    if constexpr (late_loss) {  // one more consumer barrier per row
      float wz = warp_sum(wz2.x + wz2.y);
      if (lane == 0) sh->wz[par][warp] = wz;
      ring::consumers_sync(1, NC * 32);
      if (tid == 0) {
        float t = 0.f;
        for (int c = 0; c < NC; ++c) t += sh->wz[par][c];  // fixed warp order
        const RowCoef lc = ce_row_coefs<T>(a, lse, zy, t, y);
        if (a.loss_rows) a.loss_rows[row] = lc.loss;
        if (a.z_loss_rows) a.z_loss_rows[row] = lc.zl;
      }
    }
  }
}

}  // namespace cer

int launch_ce_ring(const CeRowArgs& a, int dtype, cudaStream_t st) {
  // raw logits (standalone CE) or FLCE finalize (partials + capped logits); not vocab-parallel
  const bool part = a.partials != nullptr || a.row_stats != nullptr;  // FLCE / vocab-parallel finalize
  if (a.rows <= 0 || (part && !a.input_capped) || (!part && a.input_capped)) return LK_UNSUPPORTED;
  if (a.row_stats && (a.correct_rows || a.pred_rows)) return LK_UNSUPPORTED;
  // class weights + smoothing in the FLCE finalize need pass 2 for the weighted sum
  if (part && a.class_weight && a.label_smoothing > 0.f && (!a.compute_grad || a.row_stats)) return LK_UNSUPPORTED;
  const int64_t esz = dtype == LK_F32 ? 4 : 2;
  if ((a.n_cols * esz) % 16 || (a.ld * esz) % 16 || (reinterpret_cast<uintptr_t>(a.x) & 15)) return LK_UNSUPPORTED;
  const int stages = 6;  // 192 KB in flight per SM
  const size_t smem = (size_t)stages * cer::PIECE + 2 * stages * sizeof(uint64_t) + sizeof(cer::Smem);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(a.rows, sm_count()));
  const bool cap = a.softcap > 0.f, ls = a.label_smoothing > 0.f;
  auto go = [&](auto kern) -> int {
    LK_CUDA(ensure_smem(reinterpret_cast<const void*>(kern), (int)smem));
    kern<<<grid, cer::THREADS, smem, st>>>(a, stages);
    return check_launch("ce_ring_kernel");
  };
  const bool wls = ls && a.class_weight;
  LK_DISPATCH_FLOAT(dtype, T, {
    if (part) {
      if (wls) return cap ? go(cer::ce_ring_kernel<T, true, true, true, true>)
                          : go(cer::ce_ring_kernel<T, false, true, true, true>);
      if (cap && ls) return go(cer::ce_ring_kernel<T, true, true, true, false>);
      if (cap) return go(cer::ce_ring_kernel<T, true, false, true, false>);
      if (ls) return go(cer::ce_ring_kernel<T, false, true, true, false>);
      return go(cer::ce_ring_kernel<T, false, false, true, false>);
    }
    if (wls) return cap ? go(cer::ce_ring_kernel<T, true, true, false, true>)
                        : go(cer::ce_ring_kernel<T, false, true, false, true>);
    if (cap && ls) return go(cer::ce_ring_kernel<T, true, true, false, false>);
    if (cap) return go(cer::ce_ring_kernel<T, true, false, false, false>);
    if (ls) return go(cer::ce_ring_kernel<T, false, true, false, false>);
    return go(cer::ce_ring_kernel<T, false, false, false, false>);
  });
  return LK_OK;
}

}  // namespace lk
