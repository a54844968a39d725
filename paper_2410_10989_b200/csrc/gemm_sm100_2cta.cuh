// CTA-pair (cta_group::2) variant of the persistent tcgen05 GEMM.
//
// A cluster of two CTAs on one TPC computes a 256 x 256 tile: CTA r holds rows
// [128 r, 128 r + 128) of A and columns [128 r, 128 r + 128) of B in its own shared
// memory; the leader (rank 0) issues tcgen05.mma.cta_group::2 (M = 256, N = 256,
// K = 16), which reads the B halves of both SMs, and each CTA's TMEM receives its
// 128 x 256 slice of the accumulator.  Per SM this halves the B operand traffic
// through shared memory compared with the 1-CTA 128 x 256 tile (24 -> 16 KB of
// operand reads per 128-cycle MMA), the limit the 1-CTA kernel hits (ncu: L1/smem
// pipe ~72% busy, MMA warp starved ~37% of the time; profiles/r01_*).
//
// Synchronisation across the pair:
//   full[s]   leader-local; both CTAs' TMA (.cta_group::2) complete_tx on it
//   empty[s]  in both CTAs; the leader's tcgen05.commit multicasts to both
//   tfull[b]  in both CTAs; multicast commit after a tile's last MMA
//   tempty[b] leader-local, 8 arrivals: 4 local + 4 remote epilogue warps
//   sched ring: the leader's producer draws a tile id from the global counter,
//   stores it into both CTAs' rings (st.shared::cluster) and arrives on both sfull;
//   sempty is leader-local with 10 arrivals (MMA + 4 epilogue warps per CTA + the
//   peer's producer).
#pragma once
#include "gemm_sm100.cuh"

namespace lk {
namespace tc2 {

using tc::Args;
using tc::Problem;
constexpr int PBM = 256, PBN = 256, HALF = 128, BK = 64, STAGES = 6, SCHED = 4;
constexpr int A_BYTES = HALF * BK * 2;  // 16 KB: this CTA's 128 rows of A
constexpr int B_BYTES = HALF * BK * 2;  // 16 KB: this CTA's 128 columns of B
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_THREADS = 256;
constexpr int TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + tc::EPI_STAGING_BYTES + 1024 + 1024;

#if defined(__CUDA_ARCH__)
using tc::elect_one;
using tc::mbar_arrive;
using tc::mbar_expect_tx_addr;
using tc::mbar_init;
using tc::mbar_wait;
using tc::mbar_wait_addr;
using tc::smem_u32;
using tc::tc_fence_after;
using tc::tc_fence_before;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_2d_cg2(uint64_t map, uint32_t bar, uint32_t dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_3d_cg2(uint64_t map, uint32_t bar, uint32_t dst, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tma_4d_cg2(uint64_t map, uint32_t bar, uint32_t dst, int x, int y, int z, int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}
// One operand half-box of a k-block (CTA pair): 128 rows / columns = 2 atoms; modes as in
// Problem::a_mode (3-5 carry the piece coordinate `pc`).
__device__ __forceinline__ void load_operand2(uint64_t map, int mode, uint32_t bar, uint32_t dst, int k0, int mn0,
                                              int pc) {
  switch (mode) {
    case 0: tma_2d_cg2(map, bar, dst, k0, mn0); break;
    case 1: tma_3d_cg2(map, bar, dst, 0, k0, mn0 >> 6); break;
    case 2:
      tma_2d_cg2(map, bar, dst, mn0, k0);
      tma_2d_cg2(map, bar, dst + 8192, mn0 + 64, k0);
      break;
    case 3: tma_3d_cg2(map, bar, dst, k0, mn0, pc); break;
    case 4: tma_4d_cg2(map, bar, dst, 0, k0, mn0 >> 6, pc); break;
    default:
      tma_3d_cg2(map, bar, dst, mn0, k0, pc);
      tma_3d_cg2(map, bar, dst + 8192, mn0 + 64, k0, pc);
      break;
  }
}
__device__ __forceinline__ void umma2_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma2_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
      ::"r"(bar), "h"(mask) : "memory");
}

struct PairTile {
  int p, m_blk, n_blk;
};
// The launch's effective tile counts and K lengths: Problem::m_limit / k_limit read once per
// thread at kernel start (every role computes the same values).
struct Eff {
  int tiles0, total;
  int tm[2], kb[2];
};
__device__ __forceinline__ Eff effective(const Args& a) {
  Eff e;
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const Problem& P = a.prob[p];
    int tm = P.tiles_m, kb = P.k_blocks;
    if (p < a.n_problems) {
      if (P.m_limit) {
        int64_t lim = *P.m_limit - P.m_base;
        lim = lim < 0 ? 0 : (lim > P.M ? P.M : lim);
        tm = (int)((lim + PBM - 1) / PBM);
      }
      if (P.k_limit) {
        int64_t lim = *P.k_limit;
        lim = (lim < 1 ? 1 : lim) - P.k_base;
        lim = lim < 0 ? 0 : (lim > P.K ? P.K : lim);
        kb = (int)((lim + BK - 1) / BK);
        if (kb == 0) tm = 0;  // nothing to add (the host never limits a storing pass to zero)
      }
    }
    e.tm[p] = tm;
    e.kb[p] = kb;
  }
  e.tiles0 = e.tm[0] * a.prob[0].tiles_n;
  e.total = e.tiles0 + (a.n_problems > 1 ? e.tm[1] * a.prob[1].tiles_n : 0);
  return e;
}

__device__ __forceinline__ PairTile decode_pair(const Args& a, const Eff& e, int t) {
  PairTile c;
  c.p = (t >= e.tiles0) ? 1 : 0;
  const int lt = c.p ? t - e.tiles0 : t;
  const int tm = e.tm[c.p];
  const int tn = c.p ? a.prob[1].tiles_n : a.prob[0].tiles_n;
  const int nf = c.p ? a.prob[1].n_fast : a.prob[0].n_fast;
  if (nf) { c.n_blk = lt % tn; c.m_blk = lt / tn; }
  else { c.m_blk = lt % tm; c.n_blk = lt / tm; }
  return c;
}
#endif

template <typename T>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm2_kernel(const __grid_constant__ CUtensorMap ma0, const __grid_constant__ CUtensorMap mb0,
             const __grid_constant__ CUtensorMap ma1, const __grid_constant__ CUtensorMap mb1,
             const __grid_constant__ CUtensorMap mc0, const __grid_constant__ CUtensorMap mc1,
             const __grid_constant__ Args args) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint8_t* sStg = smem + STAGES * STAGE_BYTES;
  uint64_t* aux = reinterpret_cast<uint64_t*>(sStg + tc::EPI_STAGING_BYTES);
  uint64_t* full = aux;
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + SCHED;
  int* stile = reinterpret_cast<int*>(sempty + SCHED);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stile + SCHED);
  const Eff eff = effective(args);  // device row limits (Problem::m_limit / k_limit)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8); }
    for (int i = 0; i < SCHED; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], 10); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&ma0); tc::tma_prefetch_desc(&mb0);
    if (args.n_problems > 1) { tc::tma_prefetch_desc(&ma1); tc::tma_prefetch_desc(&mb1); }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
  const uint32_t leader_full0 = mapa(full0, 0);
  const uint32_t leader_sempty0 = mapa(smem_u32(sempty), 0);
  const uint32_t leader_tempty0 = mapa(smem_u32(tempty), 0);

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
    const uint32_t peer_stile0 = mapa(smem_u32(stile), 1), peer_sfull0 = mapa(smem_u32(sfull), 1);
    for (int it = 0;; ++it) {
      const int slot = it % SCHED;
      const uint32_t sp = (it / SCHED) & 1;
      int tile = 0;
      if (lane == 0) {
        if (leader) {
          mbar_wait(&sempty[slot], sp ^ 1);
          tile = atomicAdd(args.counter, 1);
          if (tile >= eff.total) tile = -1;
          stile[slot] = tile;
          st_cluster_u32(peer_stile0 + 4 * slot, (uint32_t)tile);
          mbar_arrive(&sfull[slot]);
          mbar_arrive_cluster(peer_sfull0 + 8 * slot);
        } else {
          mbar_wait_acq_cluster(smem_u32(&sfull[slot]), sp);
          tile = stile[slot];
          mbar_arrive_cluster(leader_sempty0 + 8 * slot);
        }
      }
      tile = __shfl_sync(0xffffffffu, tile, 0);
      if (tile < 0) break;
      const PairTile pt = decode_pair(args, eff, tile);
      const int p = pt.p;
      const int a_mode = p ? args.prob[1].a_mode : args.prob[0].a_mode;
      const int b_mode = p ? args.prob[1].b_mode : args.prob[0].b_mode;
      const int kblocks = eff.kb[p];
      const uint64_t ma = reinterpret_cast<uint64_t>(p ? &ma1 : &ma0);
      const uint64_t mb = reinterpret_cast<uint64_t>(p ? &mb1 : &mb0);
      const int m0 = pt.m_blk * PBM + (int)rank * HALF;
      const int n0 = pt.n_blk * PBN + (int)rank * HALF;
      const int kbt = p ? args.prob[1].kb_term : args.prob[0].kb_term;
      if (kbt == 0) {
        // plain K (16-bit inputs): the producer issues 2-4 TMAs per 512-cycle k-block and sits
        // on the critical path -- per-k-block work here costs the GEMM directly (a generic
        // mode switch + piece bookkeeping in this loop measured 3% slower)
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait_addr(empty0 + stage * 8, phase ^ 1);
          if (elect_one()) {
            const uint32_t fb = leader_full0 + stage * 8;
            if (leader) mbar_expect_tx_addr(full0 + stage * 8, 2 * STAGE_BYTES);
            const uint32_t a_dst = sA0 + stage * A_BYTES, b_dst = sB0 + stage * B_BYTES;
            const int k0 = kb * BK;
            if (a_mode == 0) {
              tma_2d_cg2(ma, fb, a_dst, k0, m0);
            } else if (a_mode == 1) {
              tma_3d_cg2(ma, fb, a_dst, 0, k0, m0 >> 6);
            } else {
              tma_2d_cg2(ma, fb, a_dst, m0, k0);
              tma_2d_cg2(ma, fb, a_dst + 8192, m0 + 64, k0);
            }
            if (b_mode == 0) {
              tma_2d_cg2(mb, fb, b_dst, k0, n0);
            } else if (b_mode == 1) {
              tma_3d_cg2(mb, fb, b_dst, 0, k0, n0 >> 6);
            } else {
              tma_2d_cg2(mb, fb, b_dst, n0, k0);
              tma_2d_cg2(mb, fb, b_dst + 8192, n0 + 64, k0);
            }
            // (L2 prefetch of the B operand 8/16/32 k-blocks ahead measured 5-7% slower on the
            // logits GEMM: the stall was the epilogue, not operand latency; profiles/README.md)
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      } else {
        // piece-addressed K (fp32 split operands): run `term` reads pieces pa / pb[term]
        const Problem& PP = args.prob[p];
        int term = 0, kt = 0;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait_addr(empty0 + stage * 8, phase ^ 1);
          if (elect_one()) {
            const uint32_t fb = leader_full0 + stage * 8;
            if (leader) mbar_expect_tx_addr(full0 + stage * 8, 2 * STAGE_BYTES);
            const uint32_t a_dst = sA0 + stage * A_BYTES, b_dst = sB0 + stage * B_BYTES;
            load_operand2(ma, a_mode, fb, a_dst, kt * BK, m0, PP.pa[term]);
            load_operand2(mb, b_mode, fb, b_dst, kt * BK, n0, PP.pb[term]);
          }
          if (++kt == kbt) { kt = 0; ++term; }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ===================== MMA issuer (leader CTA only) =====================
      int stage = 0;
      uint32_t phase = 0, use = 0;  // use: accumulations issued so far (TMEM buffer = use & 1)
      const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
      for (int it = 0;; ++it) {
        const int slot = it % SCHED;
        mbar_wait(&sfull[slot], (it / SCHED) & 1);
        const int tile = stile[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[slot]);
        if (tile < 0) break;
        const int p = tile >= eff.tiles0 ? 1 : 0;
        const int a_mn = tc::mode_mn(p ? args.prob[1].a_mode : args.prob[0].a_mode);
        const int b_mn = tc::mode_mn(p ? args.prob[1].b_mode : args.prob[0].b_mode);
        const int kblocks = eff.kb[p];
        const int seg_kb = args.prob[p].seg_kb > 0 ? args.prob[p].seg_kb : kblocks;
        const uint32_t idesc = p ? args.idesc[1] : args.idesc[0];
        const uint64_t a_desc0 = tc::make_desc(sA0, a_mn ? 8192u : 16u, 1024u);
        const uint64_t b_desc0 = tc::make_desc(sB0, b_mn ? 8192u : 16u, 1024u);
        const uint32_t a_k16 = a_mn ? (2048u >> 4) : (32u >> 4);
        const uint32_t b_k16 = b_mn ? (2048u >> 4) : (32u >> 4);
        int buf = 0, ks = 0;
        uint32_t d_tmem = 0;
        for (int kb = 0; kb < kblocks; ++kb) {
          if (ks == 0) {  // a new accumulation (tile, or segment of a segmented tile): next TMEM buffer
            buf = (int)(use & 1);
            mbar_wait(&tempty[buf], ((use >> 1) & 1) ^ 1);
            tc_fence_after();
            d_tmem = tmem_base + buf * PBN;
          }
          mbar_wait_addr(full0 + stage * 8, phase);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = a_desc0 + (uint64_t)((stage * A_BYTES) >> 4);
            const uint64_t bd = b_desc0 + (uint64_t)((stage * B_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma2_f16(d_tmem, ad + k * a_k16, bd + k * b_k16, idesc, (ks | k) != 0 ? 1u : 0u);
            umma2_commit_mc(empty0 + stage * 8, (uint16_t)0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (++ks == seg_kb || kb == kblocks - 1) {
            if (elect_one()) umma2_commit_mc(smem_u32(&tfull[buf]), (uint16_t)0x3);
            __syncwarp();
            ks = 0;
            ++use;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue (both CTAs) =====================
    const int q = warp & 3;
    tc::Stager sg{smem_u32(sStg) + (uint32_t)(q * 2 * tc::STG_BYTES), 0};
    uint32_t use = 0;
    for (int it = 0;; ++it) {
      const int slot = it % SCHED;
      const uint32_t sp = (it / SCHED) & 1;
      if (leader) mbar_wait(&sfull[slot], sp);
      else mbar_wait_acq_cluster(smem_u32(&sfull[slot]), sp);
      const int tile = stile[slot];
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&sempty[slot]);
        else mbar_arrive_cluster(leader_sempty0 + 8 * slot);
      }
      if (tile < 0) break;
      const PairTile pt = decode_pair(args, eff, tile);
      const Problem& P = args.prob[pt.p];
      const uint64_t omap = reinterpret_cast<uint64_t>(pt.p ? &mc1 : &mc0);
      const int row0 = pt.m_blk * PBM + (int)rank * HALF + q * 32;
      const int64_t grow = (int64_t)row0 + lane;
      const int64_t n0 = (int64_t)pt.n_blk * PBN;
      const int nseg = tc::seg_count(P);
      for (int sgi = 0; sgi < nseg; ++sgi, ++use) {
        const int buf = (int)(use & 1);
        mbar_wait(&tfull[buf], (use >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + buf * PBN + ((uint32_t)(q * 32) << 16);
        if (nseg > 1) tc::epi_segment(omap, sg, lane, row0, n0, sgi, taddr);
        else tc::run_epilogue<T>(P, omap, sg, lane, grow, row0, n0, pt.n_blk, taddr);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&tempty[buf]);
          else mbar_arrive_cluster(leader_tempty0 + 8 * buf);
        }
      }
    }
    if (lane == 0) tc::bulk_wait_all();
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
#endif
}

// kind::f16 instruction descriptor for the pair MMA (M = 256).
inline uint32_t make_idesc2(int dtype, int a_mn, int b_mn) {
  uint32_t fmt = dtype == LK_BF16 ? 1u : 0u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(PBN >> 3) << 17) | ((uint32_t)(PBM >> 4) << 24);
}

}  // namespace tc2
}  // namespace lk
