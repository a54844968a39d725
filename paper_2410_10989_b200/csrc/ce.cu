// Cross-entropy launchers, target counting, deterministic loss reduction and the
// grad_output scaling kernels used by the CE / FLCE backward.
#include "ce.cuh"

namespace lk {

__global__ void reduce_sum_kernel(const float* __restrict__ v, int64_t n, float* out) {
  // Fixed thread->element assignment and a fixed tree: bitwise deterministic
  // (the role rowfuse's math.fsum / _sequential_sum play, ops.py:556, flce.py:176-180).
  __shared__ double sh[1024];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += (double)v[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = (float)sh[0];
}

// sum_{i valid} w[y_i] in a fixed order (one CTA, double accumulation): the MEAN denominator with
// class weights (LK/ops/cross_entropy.py:369-375, sum_non_ignore_weight).
// out = sum over valid targets of w[y] (the weighted MEAN denominator); with `total`, also
// *total = sum_c w[c] over the vocabulary (the smoothing term's weight_sum).  One CTA,
// fixed-order double tree: deterministic.
__global__ void weight_sum_kernel(const int64_t* __restrict__ t, int64_t rows, int64_t ignore_index,
                                  const float* __restrict__ w, float* out, int64_t vocab, float* total) {
  __shared__ double sh[2][1024];
  double acc = 0.0, tot = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const int64_t y = t[i];
    if (y != ignore_index && y >= 0 && y < vocab) acc += (double)w[y];  // invalid targets: flagged, weight 0
  }
  if (total)
    for (int64_t c = threadIdx.x; c < vocab; c += blockDim.x) tot += (double)w[c];
  sh[0][threadIdx.x] = acc;
  sh[1][threadIdx.x] = tot;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if ((int)threadIdx.x < k) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + k];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out = (float)sh[0][0];
    if (total) *total = (float)sh[1][0];
  }
}

int launch_weight_sum(const int64_t* t, int64_t rows, int64_t ignore_index, const float* w, float* out,
                      cudaStream_t st, int64_t vocab, float* total) {
  weight_sum_kernel<<<1, 1024, 0, st>>>(t, rows, ignore_index, w, out, vocab, total);
  return check_launch("weight_sum_kernel");
}

__global__ void count_targets_kernel(const int64_t* __restrict__ t, int64_t rows, int64_t vocab,
                                     int64_t ignore_index, unsigned long long* out) {
  unsigned long long valid = 0, bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t y = t[i];
    if (y != ignore_index) {
      ++valid;
      if (y < 0 || y >= vocab) ++bad;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    valid += __shfl_xor_sync(0xffffffffu, valid, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (valid) atomicAdd(out, valid);
    if (bad) atomicAdd(out + 1, bad);
  }
}

template <typename T>
__global__ void scale_scalar_kernel(T* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                    const float* __restrict__ scale) {
  const float s = *scale;
  if (s == 1.0f) return;  // LK/ops/fused_linear_cross_entropy.py:249 skip when grad_output == 1
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, c = i - r * cols;
    T* p = x + r * ld + c;
    *p = from_f<T>(to_f<T>(*p) * s);
  }
}

template <typename T>
__global__ void scale_scalar_vec_kernel(T* __restrict__ x, int64_t n, const float* __restrict__ scale) {
  const float s = *scale;
  if (s == 1.0f) return;
  constexpr int NV = Vec16<T>::N;
  const int64_t nvec = n / NV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    Vec16<T> v;
    v.load(x + i * NV);
#pragma unroll
    for (int k = 0; k < NV; ++k) v.v[k] *= s;
    v.store(x + i * NV);
  }
  if (blockIdx.x == 0)
    for (int64_t i = nvec * NV + threadIdx.x; i < n; i += blockDim.x) x[i] = from_f<T>(to_f<T>(x[i]) * s);
}

template <typename T, typename S>
__global__ void scale_rows_kernel(T* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                  const S* __restrict__ rs) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float s = to_f<S>(rs[r]);
    T* p = x + r * ld;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) p[c] = from_f<T>(to_f<T>(p[c]) * s);
  }
}

// out[c] (+)= sum_r x[r, c] in fixed row order (grad_bias; LK/ops/fused_linear_cross_entropy.py:214-220).
template <typename T, typename O>
__global__ void colsum_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                              O* __restrict__ out, int accumulate) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float acc = accumulate ? to_f<O>(out[c]) : 0.f;
  for (int64_t r = 0; r < rows; ++r) acc += to_f<T>(x[r * ld + c]);
  out[c] = from_f<O>(acc);
}

int launch_ce_rows(const CeRowArgs& a, int dtype, cudaStream_t st) {
  if (a.rows <= 0) return LK_OK;
  LK_REQUIRE(a.rows <= 0x7fffffffLL, LK_SIZE_MISMATCH, "too many rows for one launch");
  LK_DISPATCH_FLOAT(dtype, T, {
    ce_rows_kernel<T, 512><<<(unsigned)a.rows, 512, 0, st>>>(a);
  });
  return check_launch("ce_rows_kernel");
}

int launch_count_targets(const int64_t* t, int64_t rows, int64_t vocab, int64_t ignore_index,
                         int64_t* out, cudaStream_t st) {
  LK_CUDA(cudaMemsetAsync(out, 0, 2 * sizeof(int64_t), st));
  if (rows <= 0) return LK_OK;
  int blocks = (int)std::min<int64_t>((rows + 255) / 256, 4 * sm_count());
  count_targets_kernel<<<blocks, 256, 0, st>>>(t, rows, vocab, ignore_index,
                                               reinterpret_cast<unsigned long long*>(out));
  return check_launch("count_targets_kernel");
}

int launch_reduce_sum(const float* v, int64_t n, float* out, cudaStream_t st) {
  reduce_sum_kernel<<<1, 1024, 0, st>>>(v, n, out);
  return check_launch("reduce_sum_kernel");
}

int launch_colsum_rows(const void* x, int64_t rows, int64_t cols, int64_t ld, int dtype, void* out,
                       int out_dtype, int accumulate, cudaStream_t st) {
  unsigned blocks = (unsigned)((cols + 255) / 256);
  LK_DISPATCH_FLOAT(dtype, T, {
    if (out_dtype == LK_F32)
      colsum_kernel<T, float><<<blocks, 256, 0, st>>>(static_cast<const T*>(x), rows, cols, ld,
                                                     static_cast<float*>(out), accumulate);
    else if (out_dtype == LK_BF16)
      colsum_kernel<T, __nv_bfloat16><<<blocks, 256, 0, st>>>(
          static_cast<const T*>(x), rows, cols, ld, static_cast<__nv_bfloat16*>(out), accumulate);
    else
      colsum_kernel<T, __half><<<blocks, 256, 0, st>>>(static_cast<const T*>(x), rows, cols, ld,
                                                      static_cast<__half*>(out), accumulate);
  });
  return check_launch("colsum_kernel");
}

}  // namespace lk

using namespace lk;

extern "C" size_t lk_cross_entropy_workspace_bytes(int64_t rows) {
  (void)rows;
  return 256;  // two int64 counters (n_non_ignore, out-of-range), class-weight sums at +32 / +36
}

extern "C" int lk_count_targets(const int64_t* targets, int64_t rows, int64_t vocab,
                                int64_t ignore_index, int64_t* out, void* stream) {
  LK_REQUIRE(out != nullptr, LK_INVALID_ARGUMENT, "out is null");
  LK_REQUIRE(rows == 0 || targets != nullptr, LK_INVALID_ARGUMENT, "targets is null");
  return launch_count_targets(targets, rows, vocab, ignore_index, out, as_stream(stream));
}

extern "C" int lk_cross_entropy_fwd(void* logits, int64_t ld, const int64_t* targets, int64_t rows,
                                    int64_t vocab, int dtype, int64_t ignore_index,
                                    float label_smoothing, float lse_square_scale, float softcap,
                                    int reduction, int compute_grad, float* loss_rows,
                                    float* loss_sum, float* z_loss_rows, float* z_loss_sum,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  return lk_cross_entropy_fwd_ex(logits, ld, targets, rows, vocab, dtype, ignore_index, label_smoothing,
                                 lse_square_scale, softcap, reduction, compute_grad, loss_rows, loss_sum,
                                 z_loss_rows, z_loss_sum, nullptr, nullptr, nullptr, workspace, workspace_bytes,
                                 stream);
}

extern "C" int lk_cross_entropy_fwd_ex(void* logits, int64_t ld, const int64_t* targets, int64_t rows,
                                       int64_t vocab, int dtype, int64_t ignore_index, float label_smoothing,
                                       float lse_square_scale, float softcap, int reduction, int compute_grad,
                                       float* loss_rows, float* loss_sum, float* z_loss_rows, float* z_loss_sum,
                                       float* correct_rows, int64_t* pred_rows, const float* class_weight,
                                       void* workspace, size_t workspace_bytes, void* stream) {
  LK_REQUIRE(rows >= 0 && vocab >= 1, LK_SIZE_MISMATCH, "rows must be >= 0 and vocab >= 1");
  LK_REQUIRE(ld >= vocab, LK_NON_CONTIGUOUS, "row stride smaller than vocab");
  LK_REQUIRE(rows == 0 || (logits && targets), LK_INVALID_ARGUMENT, "null logits/targets");
  LK_REQUIRE(rows == 0 || loss_rows != nullptr, LK_INVALID_ARGUMENT, "loss_rows is null");
  LK_REQUIRE(reduction >= 0 && reduction <= 2, LK_INVALID_ARGUMENT, "bad reduction");
  LK_REQUIRE(label_smoothing >= 0.f && label_smoothing <= 1.f, LK_INVALID_ARGUMENT,
             "label_smoothing must be in [0, 1]");
  LK_REQUIRE(workspace && workspace_bytes >= lk_cross_entropy_workspace_bytes(rows),
             LK_INVALID_ARGUMENT, "workspace too small");
  cudaStream_t st = as_stream(stream);
  int64_t* counts = static_cast<int64_t*>(workspace);
  float* wsum = reinterpret_cast<float*>(static_cast<char*>(workspace) + 32);
  float* wtot = reinterpret_cast<float*>(static_cast<char*>(workspace) + 36);
  const bool wls = class_weight && label_smoothing > 0.f;
  int rc = launch_count_targets(targets, rows, vocab, ignore_index, counts, st);
  if (rc) return rc;
  if (class_weight) {
    rc = launch_weight_sum(targets, rows, ignore_index, class_weight, wsum, st, vocab, wls ? wtot : nullptr);
    if (rc) return rc;
  }
  CeRowArgs a{};
  a.x = logits; a.ld = ld; a.target = targets; a.rows = rows; a.n_cols = vocab;
  a.vocab_total = vocab; a.col_offset = 0; a.ignore_index = ignore_index;
  a.label_smoothing = label_smoothing; a.lse_square_scale = lse_square_scale; a.softcap = softcap;
  a.input_capped = 0; a.reduction = reduction; a.compute_grad = compute_grad; a.n_valid = counts;
  a.loss_rows = loss_rows; a.z_loss_rows = z_loss_rows;
  a.correct_rows = correct_rows; a.pred_rows = pred_rows;
  a.class_weight = class_weight; a.sum_valid_weight = class_weight ? wsum : nullptr;
  a.weight_total = wls ? wtot : nullptr;
  // persistent TMA ring; one CTA per row (ce_rows_kernel) for shapes the ring does not take
  // (and under the LK_PATH_CE_IMPL test knob)
  rc = path_knob(LK_PATH_CE_IMPL) == 0 ? launch_ce_ring(a, dtype, st) : LK_UNSUPPORTED;
  if (rc == LK_UNSUPPORTED) rc = launch_ce_rows(a, dtype, st);
  if (rc) return rc;
  if (loss_sum) { rc = launch_reduce_sum(loss_rows, rows, loss_sum, st); if (rc) return rc; }
  if (z_loss_sum && z_loss_rows) { rc = launch_reduce_sum(z_loss_rows, rows, z_loss_sum, st); if (rc) return rc; }
  return LK_OK;
}

extern "C" int lk_scale_by_device_scalar(void* x, int64_t rows, int64_t cols, int64_t ld, int dtype,
                                         const float* scale, void* stream) {
  LK_REQUIRE(x && scale, LK_INVALID_ARGUMENT, "null pointer");
  if (rows == 0 || cols == 0) return LK_OK;
  cudaStream_t st = as_stream(stream);
  unsigned blocks = (unsigned)std::min<int64_t>((rows * cols + 2047) / 2048 + 1, 8 * sm_count());
  LK_DISPATCH_FLOAT(dtype, T, {
    if (ld == cols && (reinterpret_cast<uintptr_t>(x) & 15) == 0)
      scale_scalar_vec_kernel<T><<<blocks, 256, 0, st>>>(static_cast<T*>(x), rows * cols, scale);
    else
      scale_scalar_kernel<T><<<blocks, 256, 0, st>>>(static_cast<T*>(x), rows, cols, ld, scale);
  });
  return check_launch("scale_scalar_kernel");
}

extern "C" int lk_scale_rows(void* x, int64_t rows, int64_t cols, int64_t ld, int dtype,
                             const void* row_scale, int row_scale_dtype, void* stream) {
  LK_REQUIRE(x && row_scale, LK_INVALID_ARGUMENT, "null pointer");
  if (rows == 0 || cols == 0) return LK_OK;
  cudaStream_t st = as_stream(stream);
  unsigned blocks = (unsigned)std::min<int64_t>(rows, 65535);
  LK_DISPATCH_FLOAT(dtype, T, {
    if (row_scale_dtype == LK_F32)
      scale_rows_kernel<T, float><<<blocks, 256, 0, st>>>(static_cast<T*>(x), rows, cols, ld,
                                                         static_cast<const float*>(row_scale));
    else if (row_scale_dtype == LK_BF16)
      scale_rows_kernel<T, __nv_bfloat16><<<blocks, 256, 0, st>>>(
          static_cast<T*>(x), rows, cols, ld, static_cast<const __nv_bfloat16*>(row_scale));
    else
      scale_rows_kernel<T, __half><<<blocks, 256, 0, st>>>(static_cast<T*>(x), rows, cols, ld,
                                                          static_cast<const __half*>(row_scale));
  });
  return check_launch("scale_rows_kernel");
}

namespace lk {

template <typename T>
__global__ void __launch_bounds__(256) vp_row_stats_kernel(const T* __restrict__ x, int64_t ld, int64_t rows,
                                                           int64_t n, const int64_t* __restrict__ target,
                                                           int64_t col_offset, int64_t ignore_index,
                                                           const float4* __restrict__ partials, int64_t n_parts,
                                                           const float* __restrict__ tgt, float4* __restrict__ out) {
  __shared__ float rm[8], rs[8], rz[8];
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t y = target[row];
  if (y == ignore_index) {
    if (tid == 0) out[row] = make_float4(0.f, 1.f, 0.f, 0.f);
    return;
  }
  const int64_t yl = y - col_offset;
  float m = -INFINITY, s = 0.f, z = 0.f;
  if (partials) {
    for (int64_t j = tid; j < n_parts; j += blockDim.x) {
      float4 q = partials[row * n_parts + j];
      ms_combine(m, s, q.x, q.y);
      z += q.z;
    }
  } else {
    const T* xr = x + row * ld;
    for (int64_t i = tid; i < n; i += blockDim.x) {
      float v = to_f<T>(xr[i]);
      ms_combine(m, s, v, 1.f);
      z += v;
    }
  }
  warp_ms(m, s);
  z = warp_sum(z);
  if (lane == 0) { rm[warp] = m; rs[warp] = s; rz[warp] = z; }
  __syncthreads();
  if (warp == 0) {
    m = lane < 8 ? rm[lane] : -INFINITY;
    s = lane < 8 ? rs[lane] : 0.f;
    z = lane < 8 ? rz[lane] : 0.f;
    warp_ms(m, s);
    z = warp_sum(z);
    if (lane == 0) {
      float zt = 0.f;
      if (yl >= 0 && yl < n) zt = to_f<T>(x[row * ld + yl]);  // stored (capped, rounded) logit
      out[row] = make_float4(m, s, z, zt);
    }
  }
}

int launch_vp_row_stats(const void* x, int64_t ld, int64_t rows, int64_t n_cols, int dtype, const int64_t* target,
                        int64_t col_offset, int64_t ignore_index, const float4* partials, int64_t n_parts,
                        const float* tgt_logit, float4* out, cudaStream_t st) {
  if (rows <= 0) return LK_OK;
  LK_DISPATCH_FLOAT(dtype, T, {
    vp_row_stats_kernel<T><<<(unsigned)rows, 256, 0, st>>>(static_cast<const T*>(x), ld, rows, n_cols, target,
                                                           col_offset, ignore_index, partials, n_parts,
                                                           tgt_logit, out);
  });
  return check_launch("vp_row_stats_kernel");
}

// Vocab-parallel statistics combine: gathered[r][row] = rank r's (max, sumexp, sum_logits,
// target_logit) -> global (M, sum_r s_r exp(m_r - M), sum_r sz_r, sum_r zt_r).  Ranks are
// folded in rank order, so every rank computes bit-identical statistics from the one
// all_gather (replaces a MAX and a SUM all-reduce plus the eager rescale between them).
__global__ void __launch_bounds__(256) vp_combine_stats_kernel(const float4* __restrict__ g, int64_t world,
                                                              int64_t rows, float4* __restrict__ out) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= rows) return;
  float m = -INFINITY;
  for (int64_t r = 0; r < world; ++r) m = fmaxf(m, g[r * rows + row].x);
  float s = 0.f, sz = 0.f, zt = 0.f;
  for (int64_t r = 0; r < world; ++r) {
    const float4 q = g[r * rows + row];
    s += q.y * __expf(q.x - m);
    sz += q.z;
    zt += q.w;
  }
  out[row] = make_float4(m, s, sz, zt);
}

}  // namespace lk

extern "C" int lk_flce_vp_combine_stats(const float* gathered, int64_t world, int64_t rows, float* row_stats,
                                        void* stream) {
  LK_REQUIRE(world >= 1 && rows >= 0, LK_SIZE_MISMATCH, "world >= 1, rows >= 0 required");
  LK_REQUIRE(rows == 0 || (gathered && row_stats), LK_INVALID_ARGUMENT, "null pointer");
  if (rows == 0) return LK_OK;
  lk::vp_combine_stats_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, lk::as_stream(stream)>>>(
      reinterpret_cast<const float4*>(gathered), world, rows, reinterpret_cast<float4*>(row_stats));
  return lk::check_launch("vp_combine_stats_kernel");
}

namespace lk {

template <typename T>
__global__ void __launch_bounds__(256) cast_f32_kernel(const float* __restrict__ src, T* __restrict__ dst, int64_t n) {
  const int64_t nvec = n / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += stride) {
    float4 a, b;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(src + 8 * i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "l"(src + 8 * i + 4));
    Vec16<T> v;
    if constexpr (Vec16<T>::N == 8) {
      v.v[0] = a.x; v.v[1] = a.y; v.v[2] = a.z; v.v[3] = a.w;
      v.v[4] = b.x; v.v[5] = b.y; v.v[6] = b.z; v.v[7] = b.w;
      v.store(dst + 8 * i);
    } else {
      for (int k = 0; k < 4; ++k) { dst[8 * i + k] = from_f<T>((&a.x)[k]); dst[8 * i + 4 + k] = from_f<T>((&b.x)[k]); }
    }
  }
  for (int64_t i = nvec * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = from_f<T>(src[i]);
}

int launch_cast_f32(const float* src, void* dst, int64_t n, int dtype, cudaStream_t st) {
  if (n <= 0) return LK_OK;
  unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n / 8 + 255) / 256, 8 * (int64_t)sm_count()));
  LK_REQUIRE(((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0, LK_NON_CONTIGUOUS,
             "cast buffers must be 16-byte aligned");
  LK_DISPATCH_FLOAT(dtype, T, { cast_f32_kernel<T><<<grid, 256, 0, st>>>(src, static_cast<T*>(dst), n); });
  return check_launch("cast_f32_kernel");
}

}  // namespace lk
