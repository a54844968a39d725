// SIMT FFMA GEMM with the FLCE epilogues.
//
// This is the precision path, not the speed path: fp32 inputs must meet rtol 1e-4
// against the f64 oracle, which TF32 tensor-core math does not (SURVEY §7 "fp32
// parity": TF32 passes only 73.7% of dX elements), so fp32 FLCE runs true fp32
// FMA here.  It also serves bf16/fp16 shapes the TMA path cannot describe
// (row strides not 16-byte aligned).  bf16 at aligned shapes uses the tcgen05 GEMM.
#include "gemm_common.cuh"

namespace lk {

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

template <typename T>
__global__ void __launch_bounds__(256) simt_gemm_kernel(Operand A, Operand B, int64_t M, int64_t N,
                                                        int64_t K, EpiArgs e) {
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const T* pa = static_cast<const T*>(A.p);
  const T* pb = static_cast<const T*>(B.p);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * SG_BM, n0 = (int64_t)blockIdx.x * SG_BN;
  const bool a_kfast = A.s_k == 1, b_nfast = B.s_i == 1;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += SG_BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int el = tid + i * 256;
      int mm, kk;
      if (a_kfast) { kk = el % SG_BK; mm = el / SG_BK; } else { mm = el % SG_BM; kk = el / SG_BM; }
      int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? to_f<T>(pa[gm * A.s_i + gk * A.s_k]) : 0.f;
      int nn;
      if (b_nfast) { nn = el % SG_BN; kk = el / SG_BN; } else { kk = el % SG_BK; nn = el / SG_BK; }
      int64_t gn = n0 + nn;
      gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < K) ? to_f<T>(pb[gn * B.s_i + gk * B.s_k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t r = m0 + ty * 4 + i, c = n0 + tx * 4 + j;
      if (r < M && c < N) epi_elem(e, r, c, acc[i][j]);
    }
}

int launch_simt_gemm(const Operand& A, const Operand& B, int64_t M, int64_t N, int64_t K, int dtype,
                     const EpiArgs& e, cudaStream_t st) {
  if (M <= 0 || N <= 0) return LK_OK;
  dim3 grid((unsigned)((N + SG_BN - 1) / SG_BN), (unsigned)((M + SG_BM - 1) / SG_BM));
  LK_REQUIRE(grid.y <= 65535, LK_SIZE_MISMATCH, "SIMT GEMM: M too large");
  LK_DISPATCH_FLOAT(dtype, T, { simt_gemm_kernel<T><<<grid, 256, 0, st>>>(A, B, M, N, K, e); });
  return check_launch("simt_gemm_kernel");
}

}  // namespace lk
