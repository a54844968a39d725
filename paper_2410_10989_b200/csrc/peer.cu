// Token-sharded grad_w all-reduce over NVLink peer memory.
//
// distributed.py's token-sharded FLCE produces one partial grad_w[V, H] per rank; the
// reference's contract is that the partials add up to the unsharded dW
// (/root/reference/pkg/tests/test_flce.py:182-205).  This is that sum as one kernel over the
// ranks' symmetric buffers (CUDA IPC mappings): no NCCL, no staging copy, called per grad_w
// slice on a side stream so it overlaps the remaining slices' dW GEMMs (distributed.py).
//
// Layout of every rank's buffer: a control page (PeerCtl) then the data.  One call reduces
// the elements [offset, offset + n*esize) of every buffer:
//   1. every CTA signals ready[rank] = epoch into every peer's control page (release, system
//      scope: this rank's data is final -- the caller's stream order put the dW GEMM first);
//   2. every CTA waits until every rank signalled `epoch` into ITS control page;
//   3. rank r owns part r of the range (16-byte-aligned parts): each thread loads a 16-byte
//      vector from every rank in rank order, adds in fp32, rounds once and stores the sum into
//      every rank -- 2 (W-1)/W of the data crosses NVLink per rank, the ring all-reduce minimum;
//   4. the last CTA of the owner (ticket counter) signals done[rank] = epoch into every peer,
//      then waits until every owner signalled `epoch`, so the kernel completing means every
//      part of this rank's range holds the final sum.
// Waits poll with acquire loads and __nanosleep and give up after timeout_ns (globaltimer),
// setting the buffer's error flag: a missing peer costs a failed call, never a hung GPU.
#include "common.cuh"

namespace lk {
namespace peer {

struct PeerCtl {
  unsigned long long ready[LK_PEER_MAX];  // ready[src]: last epoch rank src signalled (data final)
  unsigned long long done[LK_PEER_MAX];   // done[src]: last epoch rank src's stores completed
  unsigned int ticket;                    // CTAs of the running call that finished their part
  unsigned int error;                     // 1 once a wait timed out
};
static_assert(sizeof(PeerCtl) <= LK_PEER_CTL_BYTES, "control page");

struct PeerArgs {
  char* base[LK_PEER_MAX];
  int rank, world;
  int64_t offset;  // bytes from each base to element 0
  int64_t n;       // elements
  int64_t part;    // elements per owner (a multiple of the 16-byte vector)
  unsigned long long epoch;
  unsigned long long timeout_ns;
};

constexpr int kThreads = 512;
constexpr int kMaxBlocks = 32;  // 32 x 512 threads x W 16-byte loads in flight: >= 2 MB at W = 8

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ PeerCtl* ctl(const PeerArgs& a, int r) { return reinterpret_cast<PeerCtl*>(a.base[r]); }

// Thread-level wait until every rank's flag (ready or done) in this rank's page reaches epoch.
__device__ bool wait_all(const PeerArgs& a, bool done_phase, unsigned long long t0) {
  PeerCtl* mine = ctl(a, a.rank);
  for (int s = 0; s < a.world; ++s) {
    const unsigned long long* f = done_phase ? &mine->done[s] : &mine->ready[s];
    while (ld_acquire(f) < a.epoch) {
      if (*reinterpret_cast<volatile unsigned int*>(&mine->error) || global_ns() - t0 > a.timeout_ns) {
        atomicExch(&mine->error, 1u);
        return false;
      }
      __nanosleep(256);
    }
  }
  return true;
}

template <typename T>
__device__ __forceinline__ T* at(const PeerArgs& a, int r) {
  return reinterpret_cast<T*>(a.base[r] + a.offset);
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads) peer_allreduce_kernel(const __grid_constant__ PeerArgs a) {
  __shared__ int ok;
  const unsigned long long t0 = global_ns();
  if (threadIdx.x < (unsigned)a.world) {  // every CTA signals (idempotent): no CTA waits on another's start
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_release(&ctl(a, threadIdx.x)->ready[a.rank], a.epoch);
  }
  if (threadIdx.x == 0) ok = wait_all(a, false, t0);
  __syncthreads();
  if (!ok) return;

  const int64_t lo = (int64_t)a.rank * a.part;
  const int64_t hi = lo + a.part < a.n ? lo + a.part : a.n;
  const int64_t tid = blockIdx.x * (int64_t)kThreads + threadIdx.x, stride = (int64_t)gridDim.x * kThreads;
  if (lo < hi) {
    if constexpr (VEC) {
      constexpr int NV = 16 / sizeof(T);
      const int64_t nv = (hi - lo) / NV;  // parts are whole vectors except the range's last one
      for (int64_t i = tid; i < nv; i += stride) {
        const int64_t e = lo + i * NV;
        uint4 raw[LK_PEER_MAX];
#pragma unroll
        for (int s = 0; s < LK_PEER_MAX; ++s)  // every rank's vector in flight before any add
          if (s < a.world) raw[s] = __ldcg(reinterpret_cast<const uint4*>(at<T>(a, s) + e));
        Vec16<T> acc;
#pragma unroll
        for (int k = 0; k < NV; ++k) acc.v[k] = 0.f;
#pragma unroll
        for (int s = 0; s < LK_PEER_MAX; ++s)  // rank order: bit-identical sums on every rank
          if (s < a.world) {
            const T* x = reinterpret_cast<const T*>(&raw[s]);
#pragma unroll
            for (int k = 0; k < NV; ++k) acc.v[k] += to_f<T>(x[k]);
          }
#pragma unroll
        for (int s = 0; s < LK_PEER_MAX; ++s)
          if (s < a.world) acc.store(at<T>(a, s) + e);
      }
      for (int64_t e = lo + nv * NV + tid; e < hi; e += stride) {  // ragged tail of the range
        float acc = 0.f;
        for (int s = 0; s < a.world; ++s) acc += to_f<T>(__ldcg(at<T>(a, s) + e));
        for (int s = 0; s < a.world; ++s) at<T>(a, s)[e] = from_f<T>(acc);
      }
    } else {
      for (int64_t e = lo + tid; e < hi; e += stride) {
        float acc = 0.f;
        for (int s = 0; s < a.world; ++s) acc += to_f<T>(__ldcg(at<T>(a, s) + e));
        for (int s = 0; s < a.world; ++s) at<T>(a, s)[e] = from_f<T>(acc);
      }
    }
  }

  // every CTA's stores, then one ticket; the last CTA publishes this owner's part as done
  __syncthreads();
  __shared__ unsigned int last;
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const unsigned int t = atomicAdd(&ctl(a, a.rank)->ticket, 1u) + 1u;
    last = t == gridDim.x;
    if (last) {
      ctl(a, a.rank)->ticket = 0u;  // calls on one buffer are stream-serialised
      asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x < (unsigned)a.world) st_release(&ctl(a, threadIdx.x)->done[a.rank], a.epoch);
  if (threadIdx.x == 0) wait_all(a, true, t0);
}

// Same blocks on every rank: the grid is a function of (part, dtype) only.
int blocks_for(int64_t part, int esize) {
  const int64_t vecs = (part * esize + 15) / 16;
  const int64_t b = (vecs + kThreads - 1) / kThreads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(kMaxBlocks, b));
}

struct DeviceScope {  // run the runtime calls on `device`, restore the caller's device
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceScope(int device) {
    cudaGetDevice(&prev);
    if (device != prev) err = cudaSetDevice(device);
  }
  ~DeviceScope() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace peer
}  // namespace lk

using namespace lk;
using namespace lk::peer;

extern "C" int lk_peer_alloc(int device, size_t data_bytes, void** base, void* ipc_handle) {
  LK_REQUIRE(base && ipc_handle, LK_INVALID_ARGUMENT, "lk_peer_alloc: null output");
  DeviceScope ds(device);
  LK_CUDA(ds.err);
  void* p = nullptr;
  LK_CUDA(cudaMalloc(&p, LK_PEER_CTL_BYTES + data_bytes));
  cudaError_t e = cudaMemset(p, 0, LK_PEER_CTL_BYTES + data_bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return fail(LK_CUDA_ERROR, std::string("lk_peer_alloc: ") + cudaGetErrorString(e));
  }
  static_assert(sizeof(cudaIpcMemHandle_t) <= LK_PEER_HANDLE_BYTES, "handle size");
  memset(ipc_handle, 0, LK_PEER_HANDLE_BYTES);
  memcpy(ipc_handle, &h, sizeof(h));
  *base = p;
  return LK_OK;
}

extern "C" int lk_peer_open(int device, const void* ipc_handle, void** base) {
  LK_REQUIRE(base && ipc_handle, LK_INVALID_ARGUMENT, "lk_peer_open: null argument");
  DeviceScope ds(device);
  LK_CUDA(ds.err);
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  LK_CUDA(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return LK_OK;
}

extern "C" int lk_peer_close(int device, void* peer_base) {
  DeviceScope ds(device);
  LK_CUDA(ds.err);
  LK_CUDA(cudaIpcCloseMemHandle(peer_base));
  return LK_OK;
}

extern "C" int lk_peer_free(int device, void* base) {
  DeviceScope ds(device);
  LK_CUDA(ds.err);
  LK_CUDA(cudaFree(base));
  return LK_OK;
}

extern "C" int lk_peer_status(int device, void* base, int clear, int* error) {
  LK_REQUIRE(base && error, LK_INVALID_ARGUMENT, "lk_peer_status: null argument");
  DeviceScope ds(device);
  LK_CUDA(ds.err);
  unsigned int* f = &reinterpret_cast<PeerCtl*>(base)->error;
  unsigned int v = 0;
  LK_CUDA(cudaMemcpy(&v, f, sizeof(v), cudaMemcpyDeviceToHost));
  // clearing also rewinds the ticket an abandoned call may have left part-counted
  if (clear && v) LK_CUDA(cudaMemset(&reinterpret_cast<PeerCtl*>(base)->ticket, 0, 2 * sizeof(unsigned int)));
  *error = (int)v;
  return LK_OK;
}

extern "C" int lk_peer_allreduce(void* const* bases, int world, int rank, int64_t offset, int64_t n, int dtype,
                                 uint64_t epoch, int64_t timeout_ns, void* stream) {
  LK_REQUIRE(bases, LK_INVALID_ARGUMENT, "lk_peer_allreduce: null bases");
  LK_REQUIRE(world >= 1 && world <= LK_PEER_MAX, LK_INVALID_ARGUMENT,
             "lk_peer_allreduce: world must be in [1, LK_PEER_MAX]");
  LK_REQUIRE(rank >= 0 && rank < world, LK_INVALID_ARGUMENT, "lk_peer_allreduce: rank out of range");
  LK_REQUIRE(dtype >= LK_F32 && dtype <= LK_F16, LK_INVALID_ARGUMENT, "lk_peer_allreduce: bad dtype");
  LK_REQUIRE(n >= 0 && epoch >= 1, LK_INVALID_ARGUMENT, "lk_peer_allreduce: n < 0 or epoch 0");
  const int esize = dtype == LK_F32 ? 4 : 2;
  LK_REQUIRE(offset >= LK_PEER_CTL_BYTES && offset % esize == 0, LK_INVALID_ARGUMENT,
             "lk_peer_allreduce: offset must lie past the control page, element-aligned");
  PeerArgs a{};
  for (int r = 0; r < world; ++r) {
    LK_REQUIRE(bases[r], LK_INVALID_ARGUMENT, "lk_peer_allreduce: null peer base");
    a.base[r] = static_cast<char*>(bases[r]);
  }
  a.rank = rank;
  a.world = world;
  a.offset = offset;
  a.n = n;
  const int64_t nv = 16 / esize;
  a.part = ((n + world - 1) / world + nv - 1) / nv * nv;
  a.epoch = epoch;
  a.timeout_ns = timeout_ns > 0 ? (unsigned long long)timeout_ns : 120ull * 1000000000ull;
  // the vector path needs every rank's range start 16-byte aligned (bases are cudaMalloc'd)
  bool vec = offset % 16 == 0;
  for (int r = 0; r < world; ++r) vec = vec && reinterpret_cast<uintptr_t>(bases[r]) % 16 == 0;
  const int blocks = blocks_for(a.part, esize);
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case LK_F32:
      if (vec) peer_allreduce_kernel<float, true><<<blocks, kThreads, 0, st>>>(a);
      else peer_allreduce_kernel<float, false><<<blocks, kThreads, 0, st>>>(a);
      break;
    case LK_BF16:
      if (vec) peer_allreduce_kernel<__nv_bfloat16, true><<<blocks, kThreads, 0, st>>>(a);
      else peer_allreduce_kernel<__nv_bfloat16, false><<<blocks, kThreads, 0, st>>>(a);
      break;
    default:
      if (vec) peer_allreduce_kernel<__half, true><<<blocks, kThreads, 0, st>>>(a);
      else peer_allreduce_kernel<__half, false><<<blocks, kThreads, 0, st>>>(a);
      break;
  }
  return check_launch("peer_allreduce_kernel");
}
