// Epilogue contract shared by the SIMT and tcgen05 GEMMs of the FLCE chunk loop.
//
// The three GEMMs of one FLCE chunk (rowfuse/flce.py:153, 160, 161-162) differ only
// in operand layout and in what happens to an output tile:
//   EPI_LOGITS : Z = X_c W^T (+bias), softcapped, rounded to the logits dtype and
//                stored into the chunk buffer; the tcgen05 path also emits per
//                (row, N-tile) online-softmax partials and captures the target logit.
//   EPI_STORE  : dX_c = alpha * dZ W, stored in the activation dtype.
//   EPI_ACCUM  : dW (+)= dZ^T X_c into an fp32 accumulator; on the last chunk the
//                sum is written straight to the weight-dtype output (final_out).
//   EPI_F32    : plain fp32 store (kernel tests).
#pragma once
#include "common.cuh"

namespace lk {

enum EpiKind { EPI_STORE = 0, EPI_ACCUM = 1, EPI_LOGITS = 2, EPI_F32 = 3 };

struct EpiArgs {
  int kind;
  int out_dtype;          // lk_dtype of `out`
  void* out;
  int64_t ldo;
  float* acc;             // EPI_ACCUM fp32 accumulator
  int64_t ldacc;
  int beta;               // EPI_ACCUM: 1 = read-modify-write, 0 = overwrite
  int final_out;          // EPI_ACCUM: write dtype(acc + tile) to `out` instead of acc
  float alpha;
  const void* bias;       // EPI_LOGITS (dtype = out_dtype)
  float softcap;          // <= 0: none
  const int64_t* target;  // EPI_LOGITS target capture (rows of this chunk)
  int64_t col_offset;     // global column of output column 0 (vocab-parallel shard)
  int64_t ignore_index;
  float4* partials;       // [M, n_parts]
  int64_t n_parts;
  float* tgt_logit;       // [M] (legacy register epilogue only)
  int want_sum;           // EPI_LOGITS: also accumulate sum of logits (label smoothing)
  int want_argmax;        // EPI_LOGITS: first column of the tile max -> partials[].w (int bits)
  int64_t M, N;           // valid output extent
};

__device__ __forceinline__ float load_any(const void* p, int64_t i, int dt) {
  if (dt == LK_F32) return static_cast<const float*>(p)[i];
  if (dt == LK_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  return __half2float(static_cast<const __half*>(p)[i]);
}
__device__ __forceinline__ void store_any(void* p, int64_t i, int dt, float v) {
  if (dt == LK_F32) static_cast<float*>(p)[i] = v;
  else if (dt == LK_BF16) static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else static_cast<__half*>(p)[i] = __float2half_rn(v);
}
__device__ __forceinline__ float round_any(float v, int dt) {
  if (dt == LK_BF16) return __bfloat162float(__float2bfloat16_rn(v));
  if (dt == LK_F16) return __half2float(__float2half_rn(v));
  return v;
}

// Scalar epilogue for one output element (SIMT path and ragged tcgen05 edges).
__device__ __forceinline__ void epi_elem(const EpiArgs& e, int64_t r, int64_t c, float v) {
  switch (e.kind) {
    case EPI_STORE:
      store_any(e.out, r * e.ldo + c, e.out_dtype, e.alpha * v);
      break;
    case EPI_ACCUM: {
      if (!e.acc) {  // accumulate in the output dtype: out = dtype(out + dtype(tile)) (Liger's order)
        const float t = round_any(v, e.out_dtype);
        store_any(e.out, r * e.ldo + c, e.out_dtype, e.beta ? load_any(e.out, r * e.ldo + c, e.out_dtype) + t : t);
        break;
      }
      float a = e.beta ? e.acc[r * e.ldacc + c] : 0.f;
      a += v;
      if (e.final_out) store_any(e.out, r * e.ldo + c, e.out_dtype, a);
      else e.acc[r * e.ldacc + c] = a;
      break;
    }
    case EPI_LOGITS: {
      if (e.bias) v += load_any(e.bias, c, e.out_dtype);
      if (e.softcap > 0.f) v = e.softcap * tanhf(v / e.softcap);
      store_any(e.out, r * e.ldo + c, e.out_dtype, v);
      break;
    }
    default:
      static_cast<float*>(e.out)[r * e.ldo + c] = v;
  }
}

// Generic-stride operand view: X(i, k) = p[i * s_i + k * s_k].
struct Operand {
  const void* p;
  int64_t s_i, s_k;
};

int launch_simt_gemm(const Operand& A, const Operand& B, int64_t M, int64_t N, int64_t K, int dtype,
                     const EpiArgs& e, cudaStream_t st);

}  // namespace lk
