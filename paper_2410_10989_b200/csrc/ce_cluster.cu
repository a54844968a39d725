// Standalone cross entropy, one HBM read + one HBM write per logit.
//
// The reference streams each row twice (statistics, then the in-place rewrite,
// rowfuse/ops.py:530-551; Liger does the same, LK/ops/cross_entropy.py:118-246).  On
// B200 a 128256-wide bf16 row (250 KB) does not fit one CTA's shared memory, so a row
// is split across a thread-block cluster of CS CTAs (CS = 1/2/4/8, <= 64 KB per CTA):
//   1. each CTA pulls its slice into shared memory with one 1D TMA bulk copy
//      (cp.async.bulk ... mbarrier::complete_tx);
//   2. local online-softmax statistics (max, sum-exp, sum of logits, target logit)
//      from shared memory, block reduction;
//   3. the CS statistics are exchanged through distributed shared memory
//      (ld.shared::cluster) and combined in rank order (deterministic);
//   4. the gradient is computed from the shared-memory copy and written once.
// Three CTAs per SM overlap one slice's load with another's store.
#include "ce.cuh"

namespace lk {
namespace cec {

constexpr int BLOCK = 512;
constexpr int64_t MAX_SLICE_BYTES = 64 * 1024;

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float4 ld_cluster_f4(const float4* local, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(s_u32(local)), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}

template <typename T>
__global__ void __launch_bounds__(BLOCK) ce_cluster_kernel(CeRowArgs a, int64_t slice, int cs) {
  constexpr int NV = Vec16<T>::N;
  constexpr bool ACC = sizeof(T) == 4;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ float4 stats;
  __shared__ float4 gstat;
  __shared__ float rm[BLOCK / 32], rsum[BLOCK / 32], rz[BLOCK / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int64_t row = blockIdx.x / cs;
  const int64_t n = a.n_cols;
  T* xrow = static_cast<T*>(a.x) + row * a.ld;
  const int64_t c0 = (int64_t)rank * slice;
  const int64_t len = c0 < n ? (n - c0 < slice ? n - c0 : slice) : 0;
  const int64_t nvec = len / NV;  // len is a multiple of NV (host check)
  const T* buf = reinterpret_cast<const T*>(sm);
  const int64_t y = a.target[row];
  const bool has_cap = a.softcap > 0.f;
  const float cap = a.softcap;

  if (y == a.ignore_index) {  // uniform over the cluster: no DSMEM traffic, no cluster barrier
    if (a.compute_grad) {
      Vec16<T> z;
#pragma unroll
      for (int e = 0; e < NV; ++e) z.v[e] = 0.f;
      for (int64_t i = tid; i < nvec; i += BLOCK) z.store(xrow + c0 + i * NV);
    }
    if (rank == 0 && tid == 0) {
      if (a.loss_rows) a.loss_rows[row] = 0.f;
      if (a.z_loss_rows) a.z_loss_rows[row] = 0.f;
    }
    return;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0 && len > 0) {
    const uint32_t bytes = (uint32_t)(len * sizeof(T));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s_u32(sm)), "l"(xrow + c0), "r"(bytes), "r"(s_u32(&bar)) : "memory");
  }
  if (len > 0) {
    uint32_t done = 0;
    do {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done) : "r"(s_u32(&bar)) : "memory");
    } while (!done);
  }
  // ---- local statistics from shared memory
  float lm = -INFINITY, ls = 0.f, lz = 0.f;
  for (int64_t i = tid; i < nvec; i += BLOCK) {
    uint4 raw = reinterpret_cast<const uint4*>(buf)[i];
    const T* e = reinterpret_cast<const T*>(&raw);
    float v[NV];
    float cm = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      v[k] = to_f<T>(e[k]);
      if (has_cap && !a.input_capped) v[k] = cap * (ACC ? tanhf(v[k] / cap) : tanh_fast(v[k] / cap));
      cm = fmaxf(cm, v[k]);
    }
    const float mn = fmaxf(lm, cm);
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) { acc += __expf(v[k] - mn); lz += v[k]; }
    ls = (lm == -INFINITY ? 0.f : ls * __expf(lm - mn)) + acc;
    lm = mn;
  }
  warp_ms(lm, ls);
  lz = warp_sum(lz);
  if (lane == 0) { rm[warp] = lm; rsum[warp] = ls; rz[warp] = lz; }
  __syncthreads();
  if (warp == 0) {
    float wm = lane < BLOCK / 32 ? rm[lane] : -INFINITY;
    float ws = lane < BLOCK / 32 ? rsum[lane] : 0.f;
    float wz = lane < BLOCK / 32 ? rz[lane] : 0.f;
    warp_ms(wm, ws);
    wz = warp_sum(wz);
    if (lane == 0) {
      const int64_t yl = y - a.col_offset - c0;
      float zt = 0.f;
      if (yl >= 0 && yl < len) {
        zt = to_f<T>(buf[yl]);
        if (has_cap && !a.input_capped) zt = cap * tanhf(zt / cap);
      }
      stats = make_float4(wm, ws, wz, zt);
    }
  }
  cluster_sync();  // every CTA's statistics are visible cluster-wide
  if (tid == 0) {
    float M = -INFINITY, S = 0.f, Z = 0.f, ZT = 0.f;
    for (int r = 0; r < cs; ++r) {
      const float4 f = ld_cluster_f4(&stats, (uint32_t)r);
      ms_combine(M, S, f.x, f.y);
      Z += f.z;
      ZT += f.w;
    }
    gstat = make_float4(M, S, Z, ZT);
  }
  cluster_sync();  // peers are done reading this CTA's stats; gstat visible in the CTA
  const float m = gstat.x, s = gstat.y, sz = gstat.z, zy = gstat.w;
  const float lse = m + logf(s);
  const float lsm = a.label_smoothing;
  const float eps = lsm / (float)a.vocab_total;
  float scale = 1.f;
  if (a.reduction == LK_REDUCTION_MEAN) {
    const int64_t nv = *a.n_valid;
    scale = 1.f / (float)(nv > 0 ? nv : 1);
  }
  if (rank == 0 && tid == 0) {
    float loss = lse - zy;
    if (lsm > 0.f) loss = loss * (1.f - lsm) + (-eps * sz + lsm * lse);
    const float zl = a.lse_square_scale * lse * lse;
    if (a.loss_rows) a.loss_rows[row] = (loss + zl) * scale;
    if (a.z_loss_rows) a.z_loss_rows[row] = zl * scale;
  }
  if (!a.compute_grad) return;
  const float inv_s = 1.f / s;
  const float zfac = 1.f + 2.f * a.lse_square_scale * lse;
  const float hit = 1.f - lsm;
  const int64_t yl = y - a.col_offset - c0;
  for (int64_t i = tid; i < nvec; i += BLOCK) {
    uint4 raw = reinterpret_cast<const uint4*>(buf)[i];
    const T* e = reinterpret_cast<const T*>(&raw);
    Vec16<T> o;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float z = to_f<T>(e[k]);
      float t = 0.f;
      if (has_cap) {
        if (a.input_capped) t = z / cap;
        else { t = ACC ? tanhf(z / cap) : tanh_fast(z / cap); z = cap * t; }
      }
      float g = __expf(z - m) * inv_s * zfac - eps;
      if (i * NV + k == yl) g -= hit;
      g *= scale;
      if (has_cap) g *= (1.f - t * t);
      o.v[k] = g;
    }
    o.store(xrow + c0 + i * NV);
  }
}

}  // namespace cec

// Returns LK_UNSUPPORTED when the shape cannot take the cluster path (caller falls back).
int launch_ce_cluster(const CeRowArgs& a, int dtype, cudaStream_t st) {
  if (a.rows <= 0 || a.partials || a.row_stats || a.correct_rows || a.pred_rows || a.class_weight ||
      a.token_scaling)
    return LK_UNSUPPORTED;
  const int64_t esz = dtype == LK_F32 ? 4 : 2;
  const int64_t nv = 16 / esz;
  if (a.n_cols % nv || a.ld % nv || (reinterpret_cast<uintptr_t>(a.x) & 15)) return LK_UNSUPPORTED;
  int cs = 1;
  while (cs < 8 && a.n_cols * esz > (int64_t)cs * cec::MAX_SLICE_BYTES) cs *= 2;
  int64_t slice = (a.n_cols + cs - 1) / cs;
  slice = (slice + nv - 1) / nv * nv;
  if (slice * esz > cec::MAX_SLICE_BYTES) return LK_UNSUPPORTED;
  if (a.rows * cs > 0x7fffffffLL) return LK_UNSUPPORTED;
  const size_t smem = (size_t)(slice * esz);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.rows * cs));
  cfg.blockDim = dim3(cec::BLOCK);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  LK_DISPATCH_FLOAT(dtype, T, {
    e = cudaFuncSetAttribute(cec::ce_cluster_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, cec::ce_cluster_kernel<T>, a, slice, cs);
  });
  if (e != cudaSuccess) return fail(LK_CUDA_ERROR, std::string("ce_cluster_kernel: ") + cudaGetErrorString(e));
  return check_launch("ce_cluster_kernel");
}

}  // namespace lk
