// Row-wise online-softmax cross entropy, gradient written in place.
//
// One kernel serves two callers:
//   * standalone CE (rowfuse/ops.py:502-560, LK/ops/cross_entropy.py:26-299):
//     pass 1 streams the row once for (max, sumexp, sum_logits); pass 2 rewrites
//     the row with d(loss)/d(logits).  Two reads + one write of the row.
//   * FLCE finalize (rowfuse/flce.py:155-157): the tcgen05 logits GEMM epilogue
//     already produced per-(row, N-tile) partial statistics, so pass 1 collapses
//     to a combine over ~V/256 partials and the row is read once and written once.
//
// Semantics follow Liger (LK/ops/cross_entropy.py:100-289): ignore_index rows get
// zero loss and zero gradient; label smoothing eps = ls / V; z-loss lse_square_scale;
// softcap cap*tanh(z/cap) with the (1 - tanh^2) chain rule; MEAN divides by the
// device-side non-ignored count.
#pragma once
#include "common.cuh"

namespace lk {

struct CeRowArgs {
  void* x;                 // [rows, ld] logits in dtype T, overwritten with grad
  int64_t ld;
  const int64_t* target;   // [rows]
  int64_t rows;
  int64_t n_cols;          // columns held in x (local vocab shard)
  int64_t vocab_total;     // V used for the smoothing eps (== n_cols unless vocab-parallel)
  int64_t col_offset;      // global column of x[:, 0] (vocab-parallel), else 0
  int64_t ignore_index;
  float label_smoothing;
  float lse_square_scale;
  float softcap;           // <= 0: none
  int input_capped;        // x already holds cap*tanh(z/cap) (FLCE epilogue output)
  int reduction;
  int compute_grad;
  const int64_t* n_valid;  // device count of non-ignored targets (MEAN)
  float* loss_rows;        // [rows] or null
  float* z_loss_rows;      // [rows] or null
  // precomputed statistics (either, or neither):
  const float4* partials;  // [rows, n_parts] (max, sumexp, sum_logits, -) per N tile
  int64_t n_parts;
  const float* tgt_logit;  // [rows] capped target logit (with partials)
  const float4* row_stats; // [rows] global (max, sumexp, sum_logits, target_logit) (vocab-parallel)
  // Liger return_token_accuracy / return_predicted_tokens (LK/ops/cross_entropy.py:131-163, 294-299):
  // argmax = first column of the (softcapped) row max; ignored rows -> 0 / -1.  With
  // partials, the argmax comes from partials[].w (int bits) written by the logits epilogue.
  float* correct_rows;     // [rows] 1.0 if argmax == target else 0.0, or null
  int64_t* pred_rows;      // [rows] argmax (global column), -1 for ignored rows, or null
  // Liger FLCE use_token_scaling (LK/ops/fused_linear_cross_entropy.py:109-139, 187-206):
  // loss, z-loss and gradient of a row scaled by its detached target probability
  // p_t = softmax(z)[t], rounded to the logits dtype as torch.softmax on the logits returns it.
  int token_scaling;
  // Liger class weights (ce_weight; LK/ops/cross_entropy.py:122-124, 220-239, 278-288), without
  // label smoothing: loss_i = w[y_i] (lse - z_y) / sum_valid(w[y]) (MEAN), gradient likewise.
  const float* class_weight;      // [vocab_total] fp32 or null
  const float* sum_valid_weight;  // device scalar sum_{valid i} w[y_i] (MEAN with class_weight)
  // class weights WITH label smoothing (LK/ops/cross_entropy.py:165-171, 227-233, 280-285):
  // smooth term eps sum_c w_c (lse - z_c); the statistics pass then sums z_c w_c, and the
  // gradient gains a per-column -eps w_c term (ce_rows_kernel only).
  const float* weight_total;      // device scalar sum_c w[c]
  // Device row limit of the kept-row FLCE (lk_flce_args.row_limit): the gradient rows of ignored
  // rows at or past round_up(max(*zero_limit, 1), 256) - zero_base are never read (the GEMMs
  // stop at that tile), so the ring kernel skips their zero writes.  null = write every row.
  const int64_t* zero_limit;
  int64_t zero_base;
};

// Per-row loss and gradient coefficients: grad = p * pc + ceps - [col == y] * chit (then the
// softcap chain rule), p = softmax(z)[col].  Reduction, token scaling and class weights fold in
// here so the streaming passes stay option-free.
struct RowCoef {
  float loss, zl, pc, ceps, chit;
};
template <typename T>
__device__ __forceinline__ RowCoef ce_row_coefs(const CeRowArgs& a, float lse, float zy, float sz, int64_t y) {
  const float lsm = a.label_smoothing, eps = lsm / (float)a.vocab_total, lss = a.lse_square_scale;
  const bool mean = a.reduction == LK_REDUCTION_MEAN;
  float inv_n = 1.f;
  if (mean) {
    const int64_t nv = *a.n_valid;
    inv_n = 1.f / (float)(nv > 0 ? nv : 1);
  }
  const float ts = a.token_scaling ? round_to<T>(__expf(zy - lse)) : 1.f;
  RowCoef c;
  if (a.class_weight) {
    // out-of-range targets (flagged by the count kernel, raised by the host) weigh 0: no OOB read
    const float wy = (y >= 0 && y < a.vocab_total) ? a.class_weight[y] : 0.f;
    float s1 = ts;
    if (mean) {
      const float swn = *a.sum_valid_weight;
      s1 = ts / (swn != 0.f ? swn : 1.f);
    }
    const float s2 = inv_n * ts;
    c.zl = lss * lse * lse * s2;
    if (lsm > 0.f) {  // sz = sum_c w_c z_c; ceps is multiplied by w[col] in the gradient pass
      const float wt = *a.weight_total;
      c.loss = ((1.f - lsm) * wy * (lse - zy) + eps * (lse * wt - sz)) * s1 + c.zl;
      c.pc = ((1.f - lsm) * wy + eps * wt) * s1 + 2.f * lss * lse * s2;
      c.ceps = -eps * s1;
      c.chit = (1.f - lsm) * wy * s1;
    } else {
      c.loss = wy * (lse - zy) * s1 + c.zl;
      c.pc = wy * s1 + 2.f * lss * lse * s2;
      c.ceps = 0.f;
      c.chit = wy * s1;
    }
  } else {
    const float rs = inv_n * ts;
    float loss = lse - zy;
    if (lsm > 0.f) loss = loss * (1.f - lsm) + (-eps * sz + lsm * lse);
    c.zl = lss * lse * lse * rs;
    c.loss = loss * rs + c.zl;
    c.pc = rs * (1.f + 2.f * lss * lse);
    c.ceps = -eps * rs;
    c.chit = (1.f - lsm) * rs;
  }
  return c;
}

// (value, index) argmax merge: larger value wins, ties keep the smaller index.
__device__ __forceinline__ void am_merge(float& v, int& i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}
__device__ __forceinline__ void warp_am(float& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    am_merge(v, i, v2, i2);
  }
}

template <typename T>
__device__ __forceinline__ float cap_val(float z, float cap, bool accurate) {
  float t = accurate ? tanhf(z / cap) : tanh_fast(z / cap);
  return cap * t;
}

template <typename T, int BLOCK>
__global__ void __launch_bounds__(BLOCK) ce_rows_kernel(CeRowArgs a) {
  constexpr int NV = Vec16<T>::N;
  constexpr bool ACCURATE = sizeof(T) == 4;
  __shared__ float red_m[BLOCK / 32], red_s[BLOCK / 32], red_z[BLOCK / 32], red_av[BLOCK / 32];
  __shared__ int red_ai[BLOCK / 32];
  __shared__ float bcast[4];
  __shared__ int bcast_arg;
  const bool want_arg = a.correct_rows || a.pred_rows;
  float av = -INFINITY;
  int ai = 0x7fffffff;

  const int64_t row = blockIdx.x;
  if (row >= a.rows) return;
  T* x = static_cast<T*>(a.x) + row * a.ld;
  const int64_t n = a.n_cols;
  const int64_t y = a.target[row];
  const bool has_cap = a.softcap > 0.f;
  const float cap = a.softcap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (y == a.ignore_index) {
    if (a.compute_grad) {
      for (int64_t i = tid; i < n; i += BLOCK) x[i] = from_f<T>(0.f);
    }
    if (tid == 0) {
      if (a.loss_rows) a.loss_rows[row] = 0.f;
      if (a.z_loss_rows) a.z_loss_rows[row] = 0.f;
      if (a.correct_rows) a.correct_rows[row] = 0.f;
      if (a.pred_rows) a.pred_rows[row] = -1;
    }
    return;
  }
  const int64_t yl = y - a.col_offset;  // local column of the target (may be outside [0, n))
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  // class weights with smoothing: the smoothing sum is sum_c w_c z_c (weights by global column)
  const float* wcol = (a.class_weight && a.label_smoothing > 0.f) ? a.class_weight + a.col_offset : nullptr;

  float m, s, sz, zy;
  if (a.row_stats) {
    float4 st = a.row_stats[row];
    m = st.x; s = st.y; sz = st.z; zy = st.w;
  } else {
    float lm = -INFINITY, ls = 0.f, lz = 0.f;
    if (a.partials) {
      const float4* p = a.partials + row * a.n_parts;
      for (int64_t j = tid; j < a.n_parts; j += BLOCK) {
        float4 q = p[j];
        ms_combine(lm, ls, q.x, q.y);
        lz += q.z;
        if (want_arg) am_merge(av, ai, q.x, __float_as_int(q.w));
      }
    } else {
      auto upd = [&](float* v, int cnt, int64_t col) {
        float cm = -INFINITY;
        for (int i = 0; i < cnt; ++i) {
          if (has_cap && !a.input_capped) v[i] = cap_val<T>(v[i], cap, ACCURATE);
          cm = fmaxf(cm, v[i]);
          if (want_arg) am_merge(av, ai, v[i], (int)(col + i));
        }
        float mn = fmaxf(lm, cm);
        float acc = 0.f;
        for (int i = 0; i < cnt; ++i) { acc += __expf(v[i] - mn); lz += wcol ? v[i] * wcol[col + i] : v[i]; }
        ls = (lm == -INFINITY ? 0.f : ls * __expf(lm - mn)) + acc;
        lm = mn;
      };
      if (vec_ok) {
        const int64_t nvec = n / NV;
        for (int64_t i = tid; i < nvec; i += BLOCK) {
          Vec16<T> v;
          v.load(x + i * NV);
          upd(v.v, NV, i * NV);
        }
        for (int64_t i = nvec * NV + tid; i < n; i += BLOCK) {
          float v = to_f<T>(x[i]);
          upd(&v, 1, i);
        }
      } else {
        for (int64_t i = tid; i < n; i += BLOCK) {
          float v = to_f<T>(x[i]);
          upd(&v, 1, i);
        }
      }
    }
    warp_ms(lm, ls);
    lz = warp_sum(lz);
    if (want_arg) warp_am(av, ai);
    if (lane == 0) { red_m[warp] = lm; red_s[warp] = ls; red_z[warp] = lz; red_av[warp] = av; red_ai[warp] = ai; }
    __syncthreads();
    if (warp == 0) {
      float wm = lane < BLOCK / 32 ? red_m[lane] : -INFINITY;
      float ws = lane < BLOCK / 32 ? red_s[lane] : 0.f;
      float wz = lane < BLOCK / 32 ? red_z[lane] : 0.f;
      float wav = lane < BLOCK / 32 ? red_av[lane] : -INFINITY;
      int wai = lane < BLOCK / 32 ? red_ai[lane] : 0x7fffffff;
      warp_ms(wm, ws);
      wz = warp_sum(wz);
      if (want_arg) {
        warp_am(wav, wai);
        if (lane == 0) bcast_arg = wai;
      }
      if (lane == 0) {
        float zt = 0.f;
        if (yl >= 0 && yl < n) {
          zt = to_f<T>(x[yl]);
          if (has_cap && !a.input_capped) zt = cap_val<T>(zt, cap, true);
        }
        bcast[0] = wm; bcast[1] = ws; bcast[2] = wz; bcast[3] = zt;
      }
    }
    __syncthreads();
    m = bcast[0]; s = bcast[1]; sz = bcast[2]; zy = bcast[3];
  }
  if (wcol && a.partials) {
    // the precomputed statistics carry the unweighted sum: one extra read of the row for
    // sum_c w_c z_c (x holds capped logits on these paths)
    float lz = 0.f;
    for (int64_t i = tid; i < n; i += BLOCK) {
      float v = to_f<T>(x[i]);
      if (has_cap && !a.input_capped) v = cap_val<T>(v, cap, ACCURATE);
      lz += v * wcol[i];
    }
    lz = warp_sum(lz);
    if (lane == 0) red_z[warp] = lz;
    __syncthreads();
    if (warp == 0) {
      float wz = lane < BLOCK / 32 ? red_z[lane] : 0.f;
      wz = warp_sum(wz);
      if (lane == 0) bcast[2] = wz;
    }
    __syncthreads();
    sz = bcast[2];
  }

  const float lse = m + logf(s);
  const RowCoef rc = ce_row_coefs<T>(a, lse, zy, sz, y);
  if (tid == 0) {
    if (want_arg) {  // global column; the finalize of a vocab shard is not supported (row_stats path)
      const int64_t am = a.row_stats ? -1 : (int64_t)bcast_arg + a.col_offset;
      if (a.pred_rows) a.pred_rows[row] = am;
      if (a.correct_rows) a.correct_rows[row] = am == y ? 1.f : 0.f;
    }
    if (a.loss_rows) a.loss_rows[row] = rc.loss;  // LK/ops/cross_entropy.py:259-289
    if (a.z_loss_rows) a.z_loss_rows[row] = rc.zl;
  }
  if (!a.compute_grad) return;

  // pass 2: d(loss)/d(z) (LK/ops/cross_entropy.py:181-246)
  const float pc = rc.pc / s;
  auto grad = [&](float z, int64_t col) -> float {
    float t = 0.f;
    if (has_cap) {
      if (a.input_capped) {
        t = z / cap;
      } else {
        t = ACCURATE ? tanhf(z / cap) : tanh_fast(z / cap);
        z = cap * t;
      }
    }
    float g = __expf(z - m) * pc + (wcol ? rc.ceps * wcol[col] : rc.ceps);
    if (col == yl) g -= rc.chit;
    if (has_cap) g *= (1.f - t * t);
    return g;
  };
  if (vec_ok) {
    const int64_t nvec = n / NV;
    for (int64_t i = tid; i < nvec; i += BLOCK) {
      Vec16<T> v;
      v.load(x + i * NV);
#pragma unroll
      for (int k = 0; k < NV; ++k) v.v[k] = grad(v.v[k], i * NV + k);
      v.store(x + i * NV);
    }
    for (int64_t i = nvec * NV + tid; i < n; i += BLOCK) x[i] = from_f<T>(grad(to_f<T>(x[i]), i));
  } else {
    for (int64_t i = tid; i < n; i += BLOCK) x[i] = from_f<T>(grad(to_f<T>(x[i]), i));
  }
}

// Deterministic fixed-order sum of n fp32 values into *out (one CTA, double accumulation).
__global__ void reduce_sum_kernel(const float* __restrict__ v, int64_t n, float* out);
// n_non_ignore and out-of-range count: out[0], out[1] (zeroed by the caller).
__global__ void count_targets_kernel(const int64_t* __restrict__ t, int64_t rows, int64_t vocab,
                                     int64_t ignore_index, unsigned long long* out);

int launch_ce_rows(const CeRowArgs& a, int dtype, cudaStream_t st);
// Persistent TMA-ring standalone CE (ce_ring.cu, default); LK_UNSUPPORTED if not applicable.
int launch_ce_ring(const CeRowArgs& a, int dtype, cudaStream_t st);
int launch_count_targets(const int64_t* t, int64_t rows, int64_t vocab, int64_t ignore_index,
                         int64_t* out, cudaStream_t st);
int launch_reduce_sum(const float* v, int64_t n, float* out, cudaStream_t st);
// sum over non-ignored rows of class_weight[target] (MEAN denominator with class weights)
int launch_weight_sum(const int64_t* t, int64_t rows, int64_t ignore_index, const float* w, float* out,
                      cudaStream_t st, int64_t vocab = 0, float* total = nullptr);
// Vocab-parallel stage 1: per-row local (max, sumexp, sum_logits, target_logit).
int launch_vp_row_stats(const void* x, int64_t ld, int64_t rows, int64_t n_cols, int dtype,
                        const int64_t* target, int64_t col_offset, int64_t ignore_index,
                        const float4* partials, int64_t n_parts, const float* tgt_logit,
                        float4* out, cudaStream_t st);
// dst[i] = dtype(src[i]) for n fp32 values (the multi-chunk dW accumulator -> grad_w).
int launch_cast_f32(const float* src, void* dst, int64_t n, int dtype, cudaStream_t st);
// fp32 -> n_terms bf16 piece copies (split.cu): dst + row*row_stride + t*term_stride + col
int launch_split_bf16(const float* src, int64_t rows, int64_t cols, int64_t ld_src, int64_t rows_pad,
                      int64_t cols_pad, void* dst, int64_t row_stride, int64_t term_stride, int n_terms,
                      const int* order, cudaStream_t st);
int launch_colsum_rows(const void* x, int64_t rows, int64_t cols, int64_t ld, int dtype,
                       void* out, int out_dtype, int accumulate, cudaStream_t st);

}  // namespace lk
