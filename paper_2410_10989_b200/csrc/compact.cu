// Row compaction around the FLCE: the rows whose target is ignore_index contribute nothing
// (loss 0, gradient row 0, no dW/db term -- rowfuse/ops.py:515-523, flce.py:161-168), so the
// host wrapper (fused_linear_cross_entropy.py) runs the chunk loop on the other rows alone and
// scatters the per-row outputs back.  10% ignored targets is 10% of the
// step's GEMM work not done.
//
//   lk_compact_rows : stable compaction map of one target vector (one CTA, block scans);
//   lk_gather_rows  : dst[i, :] = index[i] >= 0 ? src[index[i], :] : fill -- the targets'
//                     gather, the per-chunk X gather inside the FLCE (launch_gather_rows,
//                     lk_flce_args.x_row_index), and the scatter back (index = inverse map, -1
//                     for ignored rows); 16-byte vectors, one warp per wide row.
#include "common.cuh"

namespace lk {
namespace compact {

constexpr int kThreads = 1024;
constexpr int kPerThread = 8;

__global__ void __launch_bounds__(kThreads) compact_rows_kernel(const int64_t* __restrict__ t, int64_t rows,
                                                                int64_t ignore_index, int64_t* __restrict__ index,
                                                                int64_t* __restrict__ pos,
                                                                int64_t* __restrict__ count) {
  __shared__ int warp_tot[kThreads / 32];
  __shared__ int64_t carry_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t carry = 0;
  for (int64_t base = 0; base < rows; base += (int64_t)kThreads * kPerThread) {
    const int64_t r0 = base + (int64_t)threadIdx.x * kPerThread;
    bool keep[kPerThread];
    int mine = 0;
#pragma unroll
    for (int k = 0; k < kPerThread; ++k) {
      keep[k] = r0 + k < rows && t[r0 + k] != ignore_index;
      mine += keep[k];
    }
    int incl = mine;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = warp_tot[lane];
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += v;
      }
      warp_tot[lane] = wi - w;  // exclusive prefix of the warps
      if (lane == 31) carry_s = carry + wi;
    }
    __syncthreads();
    int64_t at = carry + warp_tot[warp] + (incl - mine);
#pragma unroll
    for (int k = 0; k < kPerThread; ++k) {
      if (r0 + k >= rows) break;
      if (keep[k]) {
        index[at] = r0 + k;
        pos[r0 + k] = at++;
      } else {
        pos[r0 + k] = -1;
      }
    }
    carry = carry_s;
    __syncthreads();  // warp_tot / carry_s are rewritten by the next tile
  }
  for (int64_t i = carry + threadIdx.x; i < rows; i += kThreads) index[i] = -1;
  if (threadIdx.x == 0) *count = carry;
}

// Wide rows: one warp per output row, 16-byte vectors.
__global__ void __launch_bounds__(256) gather_rows_vec_kernel(const uint4* __restrict__ src, int64_t vpr,
                                                              const int64_t* __restrict__ index, int64_t out_rows,
                                                              uint4* __restrict__ dst, uint4 fill) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < out_rows; r += warps) {
    const int64_t s = index[r];
    uint4* d = dst + r * vpr;
    if (s >= 0) {
      const uint4* p = src + s * vpr;
      int64_t v = lane;
      for (; v + 96 < vpr; v += 128) {  // four 16-byte loads in flight per lane
        const uint4 a = __ldg(p + v), b = __ldg(p + v + 32), c = __ldg(p + v + 64), e = __ldg(p + v + 96);
        d[v] = a;
        d[v + 32] = b;
        d[v + 64] = c;
        d[v + 96] = e;
      }
      for (; v < vpr; v += 32) d[v] = __ldg(p + v);
    } else {
      for (int64_t v = lane; v < vpr; v += 32) d[v] = fill;
    }
  }
}

// Anything else: one thread per element of E bytes.
template <typename E>
__global__ void gather_rows_elem_kernel(const E* __restrict__ src, int64_t cols, const int64_t* __restrict__ index,
                                        int64_t out_rows, E* __restrict__ dst, E fill) {
  const int64_t n = out_rows * cols, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / cols, c = i - r * cols;
    const int64_t s = index[r];
    dst[i] = s >= 0 ? src[s * cols + c] : fill;
  }
}

template <typename E>
int launch_elem(const void* src, int64_t cols, const int64_t* index, int64_t out_rows, void* dst, uint64_t fill,
                cudaStream_t st) {
  E f;
  memcpy(&f, &fill, sizeof(E));
  const int64_t n = out_rows * cols;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * sm_count()));
  gather_rows_elem_kernel<E><<<blocks, 256, 0, st>>>(static_cast<const E*>(src), cols, index, out_rows,
                                                     static_cast<E*>(dst), f);
  return check_launch("gather_rows_elem_kernel");
}

}  // namespace compact
}  // namespace lk

using namespace lk;
using namespace lk::compact;

extern "C" int lk_compact_rows(const int64_t* targets, int64_t rows, int64_t ignore_index, int64_t* index,
                               int64_t* pos, int64_t* count, void* stream) {
  LK_REQUIRE(rows >= 0, LK_INVALID_ARGUMENT, "lk_compact_rows: rows < 0");
  LK_REQUIRE(count && (rows == 0 || (targets && index && pos)), LK_INVALID_ARGUMENT,
             "lk_compact_rows: null pointer");
  compact_rows_kernel<<<1, kThreads, 0, as_stream(stream)>>>(targets, rows, ignore_index, index, pos, count);
  return check_launch("compact_rows_kernel");
}

namespace lk {
// dst[i, :] = index[i] >= 0 ? src[index[i], :] : fill, for i < out_rows (also used by the FLCE
// chunk loop to gather a chunk's kept X rows: lk_flce_args.x_row_index).
int launch_gather_rows(const void* src, int64_t cols, int elem_bytes, const int64_t* index, int64_t out_rows,
                       void* dst, uint64_t fill, cudaStream_t st) {
  using namespace compact;
  const int64_t row_bytes = cols * elem_bytes;
  const bool vec = row_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(dst) % 16 == 0;
  if (vec && row_bytes >= 256) {
    uint4 f;  // the fill element repeated over 16 bytes
    unsigned char* fb = reinterpret_cast<unsigned char*>(&f);
    for (int i = 0; i < 16; ++i) fb[i] = reinterpret_cast<const unsigned char*>(&fill)[i % elem_bytes];
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((out_rows + 7) / 8, 16 * sm_count()));
    gather_rows_vec_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint4*>(src), row_bytes / 16, index, out_rows,
                                                   static_cast<uint4*>(dst), f);
    return check_launch("gather_rows_vec_kernel");
  }
  switch (elem_bytes) {
    case 1: return launch_elem<uint8_t>(src, cols, index, out_rows, dst, fill, st);
    case 2: return launch_elem<uint16_t>(src, cols, index, out_rows, dst, fill, st);
    case 4: return launch_elem<uint32_t>(src, cols, index, out_rows, dst, fill, st);
    default: return launch_elem<uint64_t>(src, cols, index, out_rows, dst, fill, st);
  }
}
}  // namespace lk

extern "C" int lk_gather_rows(const void* src, int64_t cols, int elem_bytes, const int64_t* index, int64_t out_rows,
                              void* dst, uint64_t fill, void* stream) {
  LK_REQUIRE(cols >= 0 && out_rows >= 0, LK_INVALID_ARGUMENT, "lk_gather_rows: negative size");
  LK_REQUIRE(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8, LK_INVALID_ARGUMENT,
             "lk_gather_rows: elem_bytes must be 1, 2, 4 or 8");
  if (cols == 0 || out_rows == 0) return LK_OK;
  LK_REQUIRE(src && dst && index, LK_INVALID_ARGUMENT, "lk_gather_rows: null pointer");
  return launch_gather_rows(src, cols, elem_bytes, index, out_rows, dst, fill, as_stream(stream));
}
