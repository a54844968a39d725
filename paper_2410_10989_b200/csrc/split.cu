// fp32 GEMMs on the bf16 tensor cores: operand splitting for the fp32 FLCE path.
//
// An fp32 value a is split into P bf16 pieces a = a0 + a1 (+ a2) + r, each piece the bf16
// rounding of what the previous ones left (a - a0 is exact in fp32), |r| <= 2^-8P |a|.
// A product a*b is then the sum of the piece products a_i*b_j with i + j <= P - 1 (3 terms
// for P = 2, 6 for P = 3; the dropped terms are below 2^-8P relative).  Instead of a new
// GEMM kernel, the terms are laid out ALONG K: the unchanged bf16 tcgen05 GEMM runs K as
// nT = P(P+1)/2 runs, run t reading piece pa[t] of A and pb[t] of B through a trailing
// tensor-map coordinate (gemm_sm100.cuh load modes 3-5), and accumulates every term into the
// same fp32 TMEM accumulator.  Each operand is therefore split ONCE into P pieces stored
// piece-major (round 2: the first version wrote nT term copies of every operand -- and a
// second, MN-major copy of W for dX -- 2-4x the memory and split traffic; fp32 FLCE at the
// cfg2 shape went 162 -> 134 ms).  P = 3 matches fp32 products; P = 2 (~2^-16 per product)
// is available.
//
// dst(row, t, col) = piece[order[t]] of src(row, col) at dst + row*row_stride +
// t*term_stride + col, for row < rows_pad, col < cols_pad; rows >= rows or cols >= cols
// are written as zeros (the padding the K runs read must be finite).
#include "common.cuh"

namespace lk {

struct SplitArgs {
  const float* src;
  int64_t rows, cols, ld_src;
  int64_t rows_pad, cols_pad;
  __nv_bfloat16* dst;
  int64_t row_stride, term_stride;
  int n_terms, pieces;
  int order[6];
};

__device__ __forceinline__ void split3(float v, float (&p)[3]) {
  const float p0 = __bfloat162float(__float2bfloat16_rn(v));
  const float r1 = v - p0;  // exact
  const float p1 = __bfloat162float(__float2bfloat16_rn(r1));
  p[0] = p0;
  p[1] = p1;
  p[2] = r1 - p1;  // exact; rounded to bf16 at the store
}

// one thread per 4 consecutive columns of one row (16-byte load, 8-byte store per term)
__global__ void __launch_bounds__(256) split_bf16_kernel(SplitArgs a) {
  const int64_t qcols = (a.cols_pad + 3) / 4;
  const int64_t total = a.rows_pad * qcols;
  const bool vec_src = (a.ld_src % 4) == 0 && (reinterpret_cast<uintptr_t>(a.src) & 15) == 0;
  const bool vec_dst = (a.row_stride % 4) == 0 && (a.term_stride % 4) == 0 &&
                       (reinterpret_cast<uintptr_t>(a.dst) & 7) == 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / qcols;
    const int64_t c0 = (i - row * qcols) * 4;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (row < a.rows) {
      const float* s = a.src + row * a.ld_src + c0;
      if (vec_src && c0 + 4 <= a.cols) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(s));
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
      } else {
        for (int k = 0; k < 4; ++k)
          if (c0 + k < a.cols) v[k] = s[k];
      }
    }
    float p[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k) split3(v[k], p[k]);
    __nv_bfloat16* d = a.dst + row * a.row_stride + c0;
    for (int t = 0; t < a.n_terms; ++t) {
      const int o = a.order[t];
      __nv_bfloat16* dt = d + t * a.term_stride;
      if (vec_dst && c0 + 4 <= a.cols_pad) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(p[0][o], p[1][o]);
        __nv_bfloat162 hi = __floats2bfloat162_rn(p[2][o], p[3][o]);
        uint2 raw;
        raw.x = *reinterpret_cast<uint32_t*>(&lo);
        raw.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(dt) = raw;
      } else {
        for (int k = 0; k < 4; ++k)
          if (c0 + k < a.cols_pad) dt[k] = __float2bfloat16_rn(p[k][o]);
      }
    }
  }
}

int launch_split_bf16(const float* src, int64_t rows, int64_t cols, int64_t ld_src, int64_t rows_pad,
                      int64_t cols_pad, void* dst, int64_t row_stride, int64_t term_stride, int n_terms,
                      const int* order, cudaStream_t st) {
  if (rows_pad <= 0 || cols_pad <= 0) return LK_OK;
  LK_REQUIRE(n_terms >= 1 && n_terms <= 6, LK_INVALID_ARGUMENT, "1..6 split terms");
  SplitArgs a{};
  a.src = src; a.rows = rows; a.cols = cols; a.ld_src = ld_src; a.rows_pad = rows_pad; a.cols_pad = cols_pad;
  a.dst = static_cast<__nv_bfloat16*>(dst); a.row_stride = row_stride; a.term_stride = term_stride;
  a.n_terms = n_terms;
  for (int t = 0; t < n_terms; ++t) a.order[t] = order[t];
  const int64_t total = rows_pad * ((cols_pad + 3) / 4);
  const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
  split_bf16_kernel<<<blocks, 256, 0, st>>>(a);
  return check_launch("split_bf16_kernel");
}

}  // namespace lk
