// Fused linear cross entropy: chunk loop, chunk policy, workspace, TMA maps.
//
// Per chunk of rows [lo, lo + r) (rowfuse/flce.py:149-162, LK/ops/fused_linear_cross_entropy.py:96-220):
//   1. logits GEMM  Z = X_c W^T            tcgen05, epilogue: softcap, bf16 store into the
//                                          chunk buffer, per-(row, 256-col tile) online-softmax
//                                          partials, target-logit capture
//   2. finalize     dZ = softmax-grad(Z)   one read + one write of the chunk buffer (in place)
//   3. backward     dX_c = dZ W            one persistent launch with both problems,
//                   dW  (+)= dZ^T X_c      dX tiles (K = V) first, dW tiles (K = r) fill the tail
// The full BT x V logits never exist; the only vocab-sized scratch is the chunk buffer.
// MEAN divides by the device-side non-ignored count inside the finalize, so there is
// no host sync (Liger syncs on .item() at LK/ops/fused_linear_cross_entropy.py:80-81).
#include <cudaTypedefs.h>
#include <mutex>

#include "ce.cuh"
#include "gemm_sm100_2cta.cuh"

namespace lk {
namespace tc {

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool tma_ok(const TmaOperand& op) {
  return (reinterpret_cast<uintptr_t>(op.ptr) & 15) == 0 && (op.row_elems * 2) % 16 == 0 &&
         op.inner >= 1 && op.outer >= 1;
}

static bool g_allow_3d = true;  // cleared if the driver rejects the 3D MN-major map

int encode_operand(CUtensorMap* map, const TmaOperand& op, int dtype, int rows_in_box, int* mode) {
  auto enc = get_encode();
  LK_REQUIRE(enc != nullptr, LK_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  const CUtensorMapDataType dt =
      dtype == LK_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  if (op.pieces > 0) {
    // piece-addressed operand: `pieces` [outer][inner] matrices, piece_elems apart; the piece
    // is the last map coordinate (box extent 1), so a box lands exactly as modes 0 / 1 / 2 do
    LK_REQUIRE((op.piece_elems * 2) % 16 == 0, LK_INVALID_ARGUMENT, "piece stride must be 16-byte aligned");
    const cuuint64_t ps = (cuuint64_t)op.piece_elems * 2;
    CUresult r;
    if (!op.mn_major) {
      cuuint64_t dims[3] = {(cuuint64_t)op.inner, (cuuint64_t)op.outer, (cuuint64_t)op.pieces};
      cuuint64_t strides[2] = {(cuuint64_t)op.row_elems * 2, ps};
      cuuint32_t box[3] = {64u, (cuuint32_t)rows_in_box, 1u};
      r = enc(map, dt, 3, const_cast<void*>(op.ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      *mode = 3;
    } else if (op.inner % 64 == 0) {
      cuuint64_t dims[4] = {64u, (cuuint64_t)op.outer, (cuuint64_t)(op.inner / 64), (cuuint64_t)op.pieces};
      cuuint64_t strides[3] = {(cuuint64_t)op.row_elems * 2, 128u, ps};
      cuuint32_t box[4] = {64u, 64u, (cuuint32_t)(rows_in_box / 64), 1u};
      r = enc(map, dt, 4, const_cast<void*>(op.ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      *mode = 4;
    } else {
      cuuint64_t dims[3] = {(cuuint64_t)op.inner, (cuuint64_t)op.outer, (cuuint64_t)op.pieces};
      cuuint64_t strides[2] = {(cuuint64_t)op.row_elems * 2, ps};
      cuuint32_t box[3] = {64u, 64u, 1u};
      r = enc(map, dt, 3, const_cast<void*>(op.ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      *mode = 5;
    }
    LK_REQUIRE(r == CUDA_SUCCESS, LK_CUDA_ERROR, "cuTensorMapEncodeTiled (pieces) failed: " + std::to_string((int)r));
    return LK_OK;
  }
  if (op.mn_major && g_allow_3d && op.inner % 64 == 0) {
    // [K rows][MN] viewed as {64 (MN within atom), K, MN/64 atoms}: one box {64, 64, atoms}
    // lands as `atoms` contiguous 8 KB SWIZZLE_128B atoms, the UMMA MN-major canonical layout.
    cuuint64_t dims[3] = {64u, (cuuint64_t)op.outer, (cuuint64_t)(op.inner / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)op.row_elems * 2, 128u};
    cuuint32_t box[3] = {64u, 64u, (cuuint32_t)(rows_in_box / 64)};
    CUresult r = enc(map, dt, 3, const_cast<void*>(op.ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) {
      *mode = 1;
      return LK_OK;
    }
    g_allow_3d = false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)op.inner, (cuuint64_t)op.outer};
  cuuint64_t strides[1] = {(cuuint64_t)op.row_elems * 2};
  cuuint32_t box[2] = {64u, (cuuint32_t)(op.mn_major ? 64 : rows_in_box)};
  CUresult r = enc(map, dt, 2, const_cast<void*>(op.ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  LK_REQUIRE(r == CUDA_SUCCESS, LK_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  *mode = op.mn_major ? 2 : 0;
  return LK_OK;
}

// Tensor map for the epilogue's TMA store: box of 32 rows x 128 bytes, SWIZZLE_128B.
// Returns 1 if the output can take the TMA path (else the legacy register epilogue runs).
static int encode_out(CUtensorMap* map, const EpiArgs& e, int dtype) {
  const void* ptr = nullptr;
  int odt = e.out_dtype;
  int64_t ld = e.ldo;
  switch (e.kind) {
    case EPI_LOGITS:
    case EPI_STORE: ptr = e.out; break;
    case EPI_ACCUM:
      if (e.acc) { ptr = e.acc; odt = LK_F32; ld = e.ldacc; }
      else ptr = e.out;
      break;
    default: ptr = e.out; odt = LK_F32; break;
  }
  if (e.kind == EPI_ACCUM && e.acc && e.final_out) return 0;  // acc + tile -> dtype: register epilogue
  const bool is32 = (e.kind == EPI_F32) || (e.kind == EPI_ACCUM && e.acc);
  if (!ptr || e.M < 1 || e.N < 1) return 0;
  if (!is32 && odt != dtype) return 0;  // 16-bit path stores the GEMM's own dtype
  const int64_t esz = is32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * esz) % 16) return 0;
  auto enc = get_encode();
  if (!enc) return 0;
  cuuint64_t dims[2] = {(cuuint64_t)e.N, (cuuint64_t)e.M};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * esz)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), 32u};
  cuuint32_t es[2] = {1u, 1u};
  const CUtensorMapDataType dt = is32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                      : (dtype == LK_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                          : CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  CUresult r = enc(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 1 : 0;
}

// CTA-pair (cta_group::2) kernel; the single-CTA kernel only through the test knob.
int default_cta_group() { return path_knob(LK_PATH_CTA_GROUP) == 1 ? 1 : 2; }

int launch_tc_gemm(const TmaOperand* a, const TmaOperand* b, Problem* probs, int n_problems, int dtype,
                   int* counter, cudaStream_t st, int cta_group, bool register_epilogue) {
  LK_REQUIRE(dtype == LK_BF16 || dtype == LK_F16, LK_UNSUPPORTED, "tcgen05 path takes bf16/fp16");
  if (cta_group <= 0) cta_group = default_cta_group();
  const int tile_m = cta_group == 2 ? tc2::PBM : BM;
  const int b_rows_in_box = cta_group == 2 ? tc2::HALF : BN;
  CUtensorMap maps[6];
  memset(maps, 0, sizeof(maps));
  Args args;
  memset(&args, 0, sizeof(args));
  args.n_problems = n_problems;
  int total = 0;
  for (int p = 0; p < n_problems; ++p) {
    Problem& P = probs[p];
    P.tiles_m = (int)((P.M + tile_m - 1) / tile_m);
    P.tiles_n = (int)((P.N + BN - 1) / BN);
    P.k_blocks = (int)((P.K + BK - 1) / BK);
    LK_REQUIRE((a[p].pieces > 0) == (P.kb_term > 0) && (b[p].pieces > 0) == (P.kb_term > 0), LK_INVALID_ARGUMENT,
               "piece-addressed operands and Problem::kb_term go together");
    int rc = encode_operand(&maps[2 * p], a[p], dtype, BM, &P.a_mode);
    if (rc) return rc;
    rc = encode_operand(&maps[2 * p + 1], b[p], dtype, b_rows_in_box, &P.b_mode);
    if (rc) return rc;
    // LK_PATH_DW_ACCUM16 = 1: the 16-bit grad_w accumulation (later chunks) reads, adds and rounds
    // in the epilogue registers instead of a TMA reduce-add in L2
    const bool reg16 = P.epi.kind == EPI_ACCUM && !P.epi.acc && P.epi.beta && path_knob(LK_PATH_DW_ACCUM16) == 1;
    P.tma_out = (register_epilogue || reg16) ? 0 : encode_out(&maps[4 + p], P.epi, dtype);
    // segmented accumulation needs the fp32 TMA store / reduce-add epilogue
    if (P.seg_kb > 0 && (!P.tma_out || P.epi.kind != EPI_F32 || P.seg_kb >= P.k_blocks)) P.seg_kb = 0;
    args.prob[p] = P;
    args.idesc[p] = cta_group == 2 ? tc2::make_idesc2(dtype, a[p].mn_major, b[p].mn_major)
                                   : make_idesc(dtype, a[p].mn_major, b[p].mn_major);
    if (p == 0) args.tiles0 = P.tiles_m * P.tiles_n;
    total += P.tiles_m * P.tiles_n;
  }
  if (n_problems == 1) { maps[2] = maps[0]; maps[3] = maps[1]; maps[5] = maps[4]; }
  if (cta_group == 1)  // the single-CTA kernel runs every row (a limit only removes work)
    for (int p = 0; p < n_problems; ++p) { args.prob[p].m_limit = nullptr; args.prob[p].k_limit = nullptr; }
  args.total_tiles = total;
  args.counter = counter;
  if (total == 0) return LK_OK;
  // dynamic shared-memory opt-in, per device (ensure_smem caches per (kernel, device))
  cudaError_t attr_err = ensure_smem(reinterpret_cast<const void*>(gemm_kernel<__nv_bfloat16>), SMEM_BYTES);
  if (attr_err == cudaSuccess) attr_err = ensure_smem(reinterpret_cast<const void*>(gemm_kernel<__half>), SMEM_BYTES);
  if (attr_err == cudaSuccess)
    attr_err = ensure_smem(reinterpret_cast<const void*>(tc2::gemm2_kernel<__nv_bfloat16>), tc2::SMEM_BYTES);
  if (attr_err == cudaSuccess)
    attr_err = ensure_smem(reinterpret_cast<const void*>(tc2::gemm2_kernel<__half>), tc2::SMEM_BYTES);
  LK_REQUIRE(attr_err == cudaSuccess, LK_CUDA_ERROR,
             std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
  if (cta_group == 1) {
    auto kern = dtype == LK_BF16 ? gemm_kernel<__nv_bfloat16> : gemm_kernel<__half>;
    const int grid = std::min(total, sm_count());
    kern<<<grid, NUM_THREADS, SMEM_BYTES, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], args);
    return check_launch("tcgen05 gemm_kernel");
  }
  auto kern2 = dtype == LK_BF16 ? tc2::gemm2_kernel<__nv_bfloat16> : tc2::gemm2_kernel<__half>;
  const int pairs = std::min(total, sm_count() / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(tc2::NUM_THREADS);
  cfg.dynamicSmemBytes = tc2::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern2, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], args);
  if (e != cudaSuccess) return fail(LK_CUDA_ERROR, std::string("cta-pair gemm launch: ") + cudaGetErrorString(e));
  return check_launch("tcgen05 gemm2_kernel");
}

}  // namespace tc

// ------------------------------------------------------------- planning ----
static bool separate_cast() { return path_knob(LK_PATH_FLCE_SEPARATE_CAST) == 1; }

static int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}
static int64_t elt_size(int dtype) { return dtype == LK_F32 ? 4 : 2; }
static int64_t ld_logits(int64_t vocab) { return (vocab + 63) / 64 * 64; }

// Reference rule (rowfuse/flce.py:69-78):
//   C_ref = 2^ceil(log2(ceil(BT / ceil(V/H)))).
// B200 rule: at least 2048 rows per chunk when the batch has them, because every
// chunk re-streams W (V x H) through two GEMMs and costs one read-modify-write of dW;
// at C = 2048 the dW GEMM's MMA time per tile covers its RMW traffic (SURVEY §7 "hard
// parts").  Batches that would need more than LK_ACCUM_AUTO_MAX_CHUNKS 2048-row chunks
// (BT > 16384) take 4096-row chunks: half the W re-streams and dW RMWs, +3.2% at
// BT = 65536 (cfg5 at N = 1) and +0.8% at BT = 8192, for which the smaller buffer is kept
// (profiles/r02/chunk_sweep.log).  The chunk buffer is capped at 1 GiB.
int launch_gather_rows(const void* src, int64_t cols, int elem_bytes, const int64_t* index, int64_t out_rows,
                       void* dst, uint64_t fill, cudaStream_t st);  // compact.cu

static int64_t b200_chunk_rows(int64_t bt, int64_t hidden, int64_t vocab, int dtype) {
  // Fewest chunks under a row cap, split evenly in 256-row CTA-pair tiles.  Every chunk is one
  // pass of the dW GEMM over all of grad_w, and a pass costs ~0.35 ms at the Llama-3 head
  // beyond its FLOPs (measured: 4 -> 3 chunks of 8192 rows is +2.4%, 3 -> 2 is flat;
  // profiles/r02/chunk_count_probe.log), while the logits buffer grows with the chunk.
  // Cap: 3072 rows (12 tiles) up to 16384 rows, 4096 beyond, and a logits buffer <= 1.5 GiB
  // (1 GiB for fp32 inputs, whose chunk also carries three bf16 piece copies).  At the Gemma-2
  // head (V = 256000) the 1.5 GiB cap allows 3 chunks instead of 4: +1.6%
  // (profiles/r02/cfg4_chunk_ab.log).
  const int64_t ratio = (vocab + hidden - 1) / hidden;
  const int64_t c_ref = next_pow2((bt + ratio - 1) / ratio);  // the reference's rule
  const int64_t cap_bytes = dtype == LK_F32 ? (int64_t)1 << 30 : (int64_t)3 << 29;
  const int64_t row_bytes = ld_logits(vocab) * elt_size(dtype);
  const int64_t cap_rows = std::max<int64_t>(256, cap_bytes / row_bytes / 256 * 256);
  const int64_t c_max = std::min<int64_t>(bt > 2048 * LK_ACCUM_AUTO_MAX_CHUNKS ? 4096 : 3072, cap_rows);
  int64_t c;
  if (bt <= c_max) {
    c = bt;
  } else {
    const int64_t nch = (bt + c_max - 1) / c_max, tiles = (bt + 255) / 256;
    c = (tiles + nch - 1) / nch * 256;
  }
  c = std::max<int64_t>(c, std::min<int64_t>(c_ref, cap_rows));
  return std::max<int64_t>(1, std::min<int64_t>(c, std::max<int64_t>(bt, 1)));
}

struct FlceLayout {
  int64_t C, nchunks, ldz, nparts;
  bool tc, need_acc, need_bias_acc;
  // fp32 inputs on the bf16 tensor cores (split operands, csrc/split.cu)
  bool tc32;
  int pieces, nT;
  size_t off_counts, off_sched, off_z, off_parts, off_tgt, off_acc, off_bias;
  size_t off_wp, off_xp, off_dzp;  // bf16 pieces: W [P][V][H], X_c [P][C][H], dZ [P][C][ldz]
  size_t off_xg;                    // gathered X chunk [C][H] (lk_flce_args.x_row_index)
  size_t total;
};

// Term orders of the split GEMMs: term t pairs piece A_ORD[t] of X (and of W in the dX GEMM)
// with piece C_ORD[t] of W in the logits GEMM (and of dZ in both backward GEMMs); the pairs
// enumerate i + j <= pieces - 1.
static const int kOrdA2[3] = {0, 0, 1}, kOrdC2[3] = {0, 1, 0};
// k-blocks (of 64) per accumulation segment of the fp32 dX GEMM: 128 truncating K=16 MMA
// steps per segment (scripts/probe_tc_accum.py, profiles/r02_tc_accum.md)
static const int kFp32SegKb = 32;
static const int kOrdA3[6] = {0, 0, 1, 0, 1, 2}, kOrdC3[6] = {0, 1, 0, 2, 1, 0};

static bool use_tc32_path(int dtype, int64_t hidden, int force_simt) {
#ifdef LK_HAS_TCGEN05
  return dtype == LK_F32 && !force_simt && hidden % 8 == 0;
#else
  (void)dtype; (void)hidden; (void)force_simt;
  return false;
#endif
}

static bool use_tc_path(int dtype, int64_t hidden, const void* x, const void* w, int force_simt) {
#ifdef LK_HAS_TCGEN05
  if (force_simt) return false;
  if (dtype != LK_BF16 && dtype != LK_F16) return false;
  if (hidden % 8 != 0) return false;
  if (x && (reinterpret_cast<uintptr_t>(x) & 15)) return false;
  if (w && (reinterpret_cast<uintptr_t>(w) & 15)) return false;
  return true;
#else
  (void)dtype; (void)hidden; (void)x; (void)w; (void)force_simt;
  return false;
#endif
}

// Weight-dtype grad_w accumulation across chunks (LK_ACCUM_* in include/liger_b200.h).
static bool wdtype_accum(int mode, int dtype, int64_t nchunks, bool tc) {
  if (dtype == LK_F32 || nchunks <= 1 || !tc) return false;  // SIMT path keeps the fp32 accumulator
  if (mode == LK_ACCUM_WEIGHT_DTYPE) return true;
  return mode == LK_ACCUM_AUTO && nchunks <= LK_ACCUM_AUTO_MAX_CHUNKS;
}

static FlceLayout flce_layout(int64_t bt, int64_t hidden, int64_t vocab, int dtype, int64_t chunk_rows,
                              bool has_grad_w, bool has_bias_grad, bool tc, int accum_mode, bool tc32 = false,
                              int pieces = 2, bool has_grad_x = true, bool gather_x = false) {
  FlceLayout L{};
  L.tc32 = tc32;
  L.pieces = pieces == 2 ? 2 : 3;  // default 3: products exact to fp32's 2^-24
  L.nT = L.pieces == 3 ? 6 : 3;
  L.C = chunk_rows > 0 ? chunk_rows : b200_chunk_rows(bt, hidden, vocab, dtype);
  L.C = std::max<int64_t>(1, std::min<int64_t>(L.C, std::max<int64_t>(bt, 1)));
  L.nchunks = bt > 0 ? (bt + L.C - 1) / L.C : 0;
  L.ldz = ld_logits(vocab);
  L.nparts = (vocab + tc::BN - 1) / tc::BN;
  L.tc = tc;
  L.need_acc = has_grad_w && dtype != LK_F32 && L.nchunks > 1 && !wdtype_accum(accum_mode, dtype, L.nchunks, tc);
  L.need_bias_acc = has_bias_grad;
  size_t off = 0;
  auto take = [&](size_t bytes) { off = align_up(off, 1024); size_t o = off; off += bytes; return o; };
  L.off_counts = take(4 * sizeof(int64_t));  // n_valid, n_out_of_range, class-weight sum
  L.off_sched = take((size_t)(2 * L.nchunks + 2 + 16) * sizeof(int));  // + per-slice counters
  L.off_z = take((size_t)L.C * L.ldz * elt_size(dtype));
  L.off_parts = take((tc || tc32) ? (size_t)L.C * L.nparts * sizeof(float4) : 0);
  L.off_tgt = take((tc || tc32) ? (size_t)L.C * sizeof(float) : 0);
  L.off_acc = take(L.need_acc ? (size_t)vocab * hidden * sizeof(float) : 0);
  L.off_bias = take(L.need_bias_acc ? (size_t)vocab * sizeof(float) : 0);
  (void)has_grad_x;
  const size_t P = (size_t)L.pieces;
  L.off_wp = take(tc32 ? P * (size_t)vocab * hidden * 2 : 0);
  L.off_xp = take(tc32 ? P * (size_t)L.C * hidden * 2 : 0);
  L.off_dzp = take(tc32 ? P * (size_t)L.C * L.ldz * 2 : 0);
  L.off_xg = take(gather_x ? (size_t)L.C * hidden * elt_size(dtype) : 0);
  L.total = align_up(off, 1024);
  return L;
}

}  // namespace lk

using namespace lk;

extern "C" int lk_flce_plan(int64_t bt, int64_t hidden, int64_t vocab, int dtype, int64_t* chunk_rows,
                            int64_t* num_chunks) {
  LK_REQUIRE(bt >= 1 && hidden >= 1 && vocab >= 1, LK_SIZE_MISMATCH, "dimensions must be >= 1");
  int64_t c = b200_chunk_rows(bt, hidden, vocab, dtype);
  c = std::min(c, next_pow2(bt));
  if (chunk_rows) *chunk_rows = c;
  if (num_chunks) *num_chunks = (bt + c - 1) / c;
  return LK_OK;
}

extern "C" size_t lk_flce_workspace_bytes(int64_t bt, int64_t hidden, int64_t vocab, int dtype,
                                          int64_t chunk_rows, int has_grad_w) {
  bool tc = use_tc_path(dtype, hidden, nullptr, nullptr, 0);
  return flce_layout(bt, hidden, vocab, dtype, chunk_rows, has_grad_w != 0, true, tc, LK_ACCUM_AUTO,
                     use_tc32_path(dtype, hidden, 0), 0, true).total;
}

extern "C" size_t lk_flce_workspace_bytes_ex(int64_t bt, int64_t hidden, int64_t vocab, int dtype,
                                             int64_t chunk_rows, int has_grad_w, int grad_w_accum) {
  bool tc = use_tc_path(dtype, hidden, nullptr, nullptr, 0);
  return flce_layout(bt, hidden, vocab, dtype, chunk_rows, has_grad_w != 0, true, tc, grad_w_accum,
                     use_tc32_path(dtype, hidden, 0), 0, true).total;
}

static FlceLayout layout_for(const lk_flce_args* a) {
  const bool tc = use_tc_path(a->dtype, a->hidden, a->x, a->weight, a->force_simt);
  const bool tc32 = use_tc32_path(a->dtype, a->hidden, a->force_simt);
  return flce_layout(a->bt, a->hidden, a->vocab, a->dtype, a->chunk_rows, a->grad_w != nullptr,
                     a->grad_bias != nullptr, tc, a->grad_w_accum, tc32, a->fp32_pieces, a->grad_x != nullptr,
                     a->x_row_index != nullptr);
}

extern "C" size_t lk_flce_workspace_bytes_for(const lk_flce_args* a) {
  if (!a) return 0;
  return layout_for(a).total;
}

extern "C" int lk_flce_forward_backward(const lk_flce_args* a) {
  LK_REQUIRE(a != nullptr, LK_INVALID_ARGUMENT, "args is null");
  const int64_t BT = a->bt, H = a->hidden, V = a->vocab;
  const int dt = a->dtype;
  LK_REQUIRE(BT >= 0 && H >= 1 && V >= 1, LK_SIZE_MISMATCH, "bt >= 0, hidden >= 1, vocab >= 1 required");
  LK_REQUIRE(dt == LK_F32 || dt == LK_BF16 || dt == LK_F16, LK_INVALID_ARGUMENT, "unknown dtype");
  LK_REQUIRE(a->reduction >= 0 && a->reduction <= 2, LK_INVALID_ARGUMENT, "bad reduction");
  LK_REQUIRE(a->label_smoothing >= 0.f && a->label_smoothing <= 1.f, LK_INVALID_ARGUMENT,
             "label_smoothing must be in [0, 1]");
  LK_REQUIRE(a->bt == 0 || a->loss_rows != nullptr, LK_INVALID_ARGUMENT, "loss_rows is null");
  LK_REQUIRE(BT == 0 || (a->x && a->weight && a->target), LK_INVALID_ARGUMENT, "null input");
  cudaStream_t st = as_stream(a->stream);
  const bool tc = use_tc_path(dt, H, a->x, a->weight, a->force_simt);
  const bool want_grad = a->grad_x || a->grad_w || a->grad_bias;
  LK_REQUIRE(a->grad_w_accum >= LK_ACCUM_AUTO && a->grad_w_accum <= LK_ACCUM_WEIGHT_DTYPE, LK_INVALID_ARGUMENT,
             "bad grad_w_accum");
  LK_REQUIRE(a->fp32_pieces == 0 || a->fp32_pieces == 2 || a->fp32_pieces == 3, LK_INVALID_ARGUMENT,
             "fp32_pieces must be 0 (default), 2 or 3");
  FlceLayout L = layout_for(a);
  const bool tc32 = L.tc32;
  const bool wacc = a->grad_w && wdtype_accum(a->grad_w_accum, dt, L.nchunks, tc);
  LK_REQUIRE(a->workspace && a->workspace_bytes >= L.total, LK_INVALID_ARGUMENT,
             "workspace too small: need " + std::to_string(L.total) + " bytes");
  char* ws = static_cast<char*>(a->workspace);
  // fp32 inputs: each operand is split ONCE into P bf16 pieces, stored piece-major; the GEMMs
  // address the piece of each K run through a trailing tensor-map coordinate (load modes 3-5),
  // so the term products i + j <= P - 1 need no duplicated copies
  const int* ordA = L.pieces == 3 ? kOrdA3 : kOrdA2;  // piece of the left operand per term
  const int* ordC = L.pieces == 3 ? kOrdC3 : kOrdC2;  // piece of the right operand per term
  const int64_t nT = L.nT, NP = L.pieces;
  static const int kIdent[3] = {0, 1, 2};
  void* wp = ws + L.off_wp;    // W pieces    [P][V][H]:   logits B (K-major), dX B (MN-major, K = v)
  void* xp = ws + L.off_xp;    // X_c pieces  [P][C][H]:   logits A (K-major), dW B (MN-major, K = row)
  void* dzp = ws + L.off_dzp;  // dZ pieces   [P][C][ldz]: dX A (K-major, K = v), dW A (MN-major, K = row)
  auto set_terms = [&](tc::Problem& Pr, int64_t k_run) {  // K = nT runs of ceil(k_run / 64) k-blocks
    Pr.kb_term = (int)((k_run + tc::BK - 1) / tc::BK);
    Pr.K = nT * Pr.kb_term * tc::BK;
    for (int t = 0; t < nT; ++t) { Pr.pa[t] = (unsigned char)ordA[t]; Pr.pb[t] = (unsigned char)ordC[t]; }
  };
  int64_t* counts = reinterpret_cast<int64_t*>(ws + L.off_counts);
  int* sched = reinterpret_cast<int*>(ws + L.off_sched);
  void* zbuf = ws + L.off_z;
  float4* parts = reinterpret_cast<float4*>(ws + L.off_parts);
  float* tgt = reinterpret_cast<float*>(ws + L.off_tgt);
  float* dwacc = reinterpret_cast<float*>(ws + L.off_acc);
  float* bacc = reinterpret_cast<float*>(ws + L.off_bias);
  const int64_t es = elt_size(dt);

  int rc;
  {
    ProfScope ps(3, st);
    rc = launch_count_targets(a->target, BT, V, a->ignore_index, counts, st);
  }
  if (rc) return rc;
  if (a->target_stats)
    LK_CUDA(cudaMemcpyAsync(a->target_stats, counts, 2 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  LK_REQUIRE(!a->ce_weight || !a->mean_count || a->mean_weight_sum || a->reduction != LK_REDUCTION_MEAN,
             LK_INVALID_ARGUMENT, "token-sharded MEAN with ce_weight needs the global weight sum (mean_weight_sum)");
  const bool wls = a->ce_weight && a->label_smoothing > 0.f;
  if (a->ce_weight && BT > 0) {  // MEAN denominator: sum of the valid targets' weights (after counts)
    rc = launch_weight_sum(a->target, BT, a->ignore_index, a->ce_weight, reinterpret_cast<float*>(counts + 2), st,
                           V, wls ? reinterpret_cast<float*>(counts + 3) : nullptr);
    if (rc) return rc;
  }
  if (tc || tc32) LK_CUDA(cudaMemsetAsync(sched, 0, (size_t)(2 * L.nchunks + 2 + 16) * sizeof(int), st));
  // grad_w slice events: the caller all-reduces slice s once event s fires, so EVERY event is
  // recorded on `st` after the work that finalises its rows on every path (sliced tcgen05 last
  // chunk: after each slice; otherwise -- SIMT, BT == 0, unsupported slice counts -- after all
  // of grad_w is written).  Slicing itself needs 2..LK_MAX_GRAD_W_SLICES slices.
  const int n_events = a->grad_w_slice_events ? std::max(0, a->grad_w_slices) : 0;
  int recorded = 0;
  auto record_rest = [&]() -> int {
    for (; recorded < n_events; ++recorded)
      LK_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(a->grad_w_slice_events[recorded]), st));
    return LK_OK;
  };
  if (BT == 0) {
    if (a->loss_sum) LK_CUDA(cudaMemsetAsync(a->loss_sum, 0, sizeof(float), st));
    if (a->z_loss_sum) LK_CUDA(cudaMemsetAsync(a->z_loss_sum, 0, sizeof(float), st));
    if (a->grad_w) LK_CUDA(cudaMemsetAsync(a->grad_w, 0, (size_t)V * H * es, st));
    if (a->grad_bias) LK_CUDA(cudaMemsetAsync(a->grad_bias, 0, (size_t)V * es, st));
    return record_rest();
  }

  if (tc32) {  // split W once per call into its P pieces
    ProfScope ps(3, st);
    rc = launch_split_bf16(static_cast<const float*>(a->weight), V, H, H, V, H, wp, H, V * H, (int)NP, kIdent, st);
    if (rc) return rc;
  }

  for (int64_t ci = 0; ci < L.nchunks; ++ci) {
    const int64_t lo = ci * L.C;
    const int64_t r = std::min(L.C, BT - lo);
    const char* xc = static_cast<const char*>(a->x) + lo * H * es;
    if (a->x_row_index) {  // kept-row gather: this chunk's X rows into the chunk-sized buffer
      ProfScope ps(3, st);
      char* xg = ws + L.off_xg;
      rc = launch_gather_rows(a->x, H, (int)es, a->x_row_index + lo, r, xg, 0, st);
      if (rc) return rc;
      xc = xg;
    }
    const bool first = ci == 0, last = ci == L.nchunks - 1;
    if (tc32) {
      ProfScope ps(3, st);
      rc = launch_split_bf16(reinterpret_cast<const float*>(xc), r, H, H, r, H, xp, H, L.C * H, (int)NP, kIdent, st);
      if (rc) return rc;
    }

    // ---- 1. logits ----
    EpiArgs le{};
    le.kind = EPI_LOGITS; le.out_dtype = dt; le.out = zbuf; le.ldo = L.ldz; le.alpha = 1.f;
    le.bias = a->bias; le.softcap = a->softcap; le.target = a->target + lo; le.col_offset = 0;
    le.ignore_index = a->ignore_index; le.partials = parts; le.n_parts = L.nparts; le.tgt_logit = tgt;
    le.M = r; le.N = V; le.want_sum = a->label_smoothing > 0.f ? 1 : 0;
    le.want_argmax = (a->token_correct_rows || a->predicted_tokens) ? 1 : 0;
    {
      ProfScope ps(0, st);
      if (tc) {
        tc::TmaOperand A{xc, H, r, H, 0}, B{a->weight, H, V, H, 0};
        tc::Problem P{};
        // m-fastest raster: the 8 pairs working on one W tile run together (W read once from HBM;
        // n-fastest measured 15% slower, profiles/README.md)
        P.M = r; P.N = V; P.K = H; P.n_fast = 0; P.epi = le;
        P.m_limit = a->row_limit; P.m_base = lo;
        rc = tc::launch_tc_gemm(&A, &B, &P, 1, dt, sched + 2 * ci, st);
      } else if (tc32) {  // fp32 logits = sum over the terms of X piece ordA[t] . W piece ordC[t]
        tc::TmaOperand A{xp, H, r, H, 0, (int)NP, L.C * H}, B{wp, H, V, H, 0, (int)NP, V * H};
        tc::Problem P{};
        P.M = r; P.N = V; P.n_fast = 0; P.epi = le;
        P.m_limit = a->row_limit; P.m_base = lo;
        set_terms(P, H);
        rc = tc::launch_tc_gemm(&A, &B, &P, 1, LK_BF16, sched + 2 * ci, st);
      } else {
        Operand A{xc, H, 1}, B{a->weight, H, 1};
        rc = launch_simt_gemm(A, B, r, V, H, dt, le, st);
      }
    }
    if (rc) return rc;

    // ---- 2. finalize: loss rows + dZ in place ----
    CeRowArgs ce{};
    ce.x = zbuf; ce.ld = L.ldz; ce.target = a->target + lo; ce.rows = r; ce.n_cols = V; ce.vocab_total = V;
    ce.col_offset = 0; ce.ignore_index = a->ignore_index; ce.label_smoothing = a->label_smoothing;
    ce.lse_square_scale = a->lse_square_scale; ce.softcap = a->softcap; ce.input_capped = 1;
    ce.reduction = a->reduction; ce.compute_grad = want_grad ? 1 : 0;
    ce.n_valid = a->mean_count ? a->mean_count : counts;
    ce.loss_rows = a->loss_rows + lo; ce.z_loss_rows = a->z_loss_rows ? a->z_loss_rows + lo : nullptr;
    ce.correct_rows = a->token_correct_rows ? a->token_correct_rows + lo : nullptr;
    ce.token_scaling = a->use_token_scaling;
    ce.class_weight = a->ce_weight;
    ce.sum_valid_weight = !a->ce_weight ? nullptr
                          : a->mean_weight_sum ? a->mean_weight_sum : reinterpret_cast<const float*>(counts + 2);
    ce.weight_total = wls ? reinterpret_cast<const float*>(counts + 3) : nullptr;
    ce.pred_rows = a->predicted_tokens ? a->predicted_tokens + lo : nullptr;
    // unread rows only when every reader stops at the limit: the tcgen05 dX GEMM (M tiles), the
    // dW GEMM (K loop: not in a last chunk that folds the fp32 accumulator, which reads every
    // row) and no bias column sum (reads every row)
    // (and only on the CTA-pair GEMM: the single-CTA test path ignores limits)
    if (a->row_limit && tc && tc::default_cta_group() == 2 && !a->grad_bias && !(a->grad_w && last && L.need_acc)) {
      ce.zero_limit = a->row_limit;
      ce.zero_base = lo;
    }
    if (tc || tc32) { ce.partials = parts; ce.n_parts = L.nparts; ce.tgt_logit = tgt; }
    {
      ProfScope ps(1, st);
      rc = (tc || tc32) && path_knob(LK_PATH_FLCE_FINALIZE) == 0 ? launch_ce_ring(ce, dt, st) : LK_UNSUPPORTED;
      if (rc == LK_UNSUPPORTED) rc = launch_ce_rows(ce, dt, st);
    }
    if (rc) return rc;
    if (!want_grad) continue;

    if (a->grad_bias) {
      ProfScope ps(3, st);
      rc = launch_colsum_rows(zbuf, r, V, L.ldz, dt, bacc, LK_F32, first ? 0 : 1, st);
      if (rc) return rc;
    }

    // ---- 3. dX = dZ W, dW (+)= dZ^T X ----
    EpiArgs xe{};
    xe.kind = EPI_STORE; xe.out_dtype = dt; xe.out = a->grad_x ? static_cast<char*>(a->grad_x) + lo * H * es : nullptr;
    xe.ldo = H; xe.alpha = 1.f; xe.M = r; xe.N = H;
    // dW: one chunk -> written straight to grad_w; several chunks -> fp32 accumulator
    // (first chunk stores, later chunks reduce-add in L2 via TMA), cast to grad_w after
    // the loop.  fp32 weights accumulate in grad_w itself.
    EpiArgs we{};
    we.kind = EPI_ACCUM; we.out_dtype = dt; we.out = a->grad_w; we.ldo = H; we.M = V; we.N = H; we.alpha = 1.f;
    if (dt == LK_F32) {
      we.acc = static_cast<float*>(a->grad_w); we.ldacc = H; we.beta = first ? 0 : 1; we.final_out = 0;
    } else if (L.nchunks == 1) {
      we.acc = nullptr; we.ldacc = H; we.beta = 0; we.final_out = 1;
    } else if (wacc) {
      // accumulate in the weight dtype inside grad_w: first chunk stores, later chunks
      // TMA reduce-add (bf16/fp16 add in L2) -- Liger's accum_dtype=None order
      we.acc = nullptr; we.ldacc = H; we.beta = first ? 0 : 1; we.final_out = 0;
    } else {
      // last chunk: grad_w = dtype(acc + tile) straight from the epilogue (register path),
      // instead of a TMA reduce-add into acc and a separate cast pass: -3.15 GB of HBM
      // traffic at cfg2 (the LK_PATH_FLCE_SEPARATE_CAST test knob restores the old order)
      const bool fold = last && !separate_cast();
      we.acc = dwacc; we.ldacc = H; we.beta = first ? 0 : 1; we.final_out = fold ? 1 : 0;
    }
    if (tc32) {  // dZ (fp32, in the chunk buffer) -> its P pieces, zero-padded to ldz columns
      ProfScope ps(3, st);
      rc = launch_split_bf16(static_cast<const float*>(zbuf), r, V, L.ldz, r, L.ldz, dzp, L.ldz, L.C * L.ldz,
                             (int)NP, kIdent, st);
      if (rc) return rc;
      xe.kind = EPI_F32;  // dX in fp32 straight from the accumulator
    }
    ProfScope ps_bwd(2, st);
    if (tc || tc32) {
      const int gdt = tc32 ? LK_BF16 : dt;
      // operands of the two backward problems: the bf16 chunk / X for 16-bit inputs; for fp32
      // inputs the piece-major dZ / W / X pieces, K = nT runs (dX: ldz per run, dW: r per run)
      const int npc = tc32 ? (int)NP : 0;
      const tc::TmaOperand dxA = tc32 ? tc::TmaOperand{dzp, L.ldz, r, L.ldz, 0, npc, L.C * L.ldz}
                                      : tc::TmaOperand{zbuf, V, r, L.ldz, 0};
      const tc::TmaOperand dxB = tc32 ? tc::TmaOperand{wp, H, V, H, 1, npc, V * H} : tc::TmaOperand{a->weight, H, V, H, 1};
      // dW K loop stops at the device row limit, except on the split-operand path (K is runs of
      // pieces) and in a last chunk that must write grad_w from the fp32 accumulator (a pass
      // limited to zero rows would skip that write)
      const bool dw_k_limit = a->row_limit && !tc32 && !(last && L.need_acc);
      const void* dwA_base = tc32 ? dzp : zbuf;
      const void* dwB_base = tc32 ? xp : xc;
      auto dw_ops = [&](int64_t v0, int64_t v1, tc::TmaOperand& A, tc::TmaOperand& B) {
        A = tc::TmaOperand{static_cast<const char*>(dwA_base) + v0 * (tc32 ? 2 : es), v1 - v0, r, L.ldz, 1, npc,
                           L.C * L.ldz};
        B = tc::TmaOperand{dwB_base, H, r, H, 1, npc, L.C * H};
      };
      tc::TmaOperand As[2], Bs[2];
      tc::Problem Ps[2];
      int np = 0;
      if (a->grad_x) {
        As[np] = dxA;
        Bs[np] = dxB;
        Ps[np] = tc::Problem{};
        Ps[np].M = r; Ps[np].N = H; Ps[np].K = V; Ps[np].n_fast = 0; Ps[np].epi = xe;
        Ps[np].m_limit = a->row_limit; Ps[np].m_base = lo;
        if (tc32) {
          set_terms(Ps[np], L.ldz);
          // fp32 dX (K = nT x ldz): restart the truncating tensor-core accumulation every
          // kFp32SegKb k-blocks and add the segments in fp32 (Problem::seg_kb)
          Ps[np].seg_kb = kFp32SegKb;
        }
        ++np;
      }
      const int slices =
          (last && a->grad_w && n_events >= 2 && n_events <= LK_MAX_GRAD_W_SLICES) ? n_events : 1;
      if (a->grad_w && slices <= 1) {
        dw_ops(0, V, As[np], Bs[np]);
        Ps[np] = tc::Problem{};
        Ps[np].M = V; Ps[np].N = H; Ps[np].K = r; Ps[np].n_fast = 1; Ps[np].epi = we;
        if (tc32) set_terms(Ps[np], r);
        if (dw_k_limit) { Ps[np].k_limit = a->row_limit; Ps[np].k_base = lo; }
        ++np;
      }
      if (np) rc = tc::launch_tc_gemm(As, Bs, Ps, np, gdt, sched + 2 * ci + 1, st);
      // token-sharded overlap: the last chunk's dW in vocab-row slices, one event per slice
      const int64_t step = (V + slices - 1) / slices;
      const int64_t sl_rows = (step + 255) / 256 * 256;
      for (int sl = 0; !rc && slices > 1 && sl < slices; ++sl) {
        const int64_t v0 = sl * sl_rows, v1 = std::min<int64_t>(V, v0 + sl_rows);
        if (v0 < v1) {
          EpiArgs ws = we;
          ws.out = static_cast<char*>(a->grad_w) + v0 * H * es;
          if (ws.acc) ws.acc = ws.acc + v0 * H;
          ws.M = v1 - v0;
          tc::TmaOperand As1, Bs1;
          dw_ops(v0, v1, As1, Bs1);
          tc::Problem P1{};
          P1.M = v1 - v0; P1.N = H; P1.K = r; P1.n_fast = 1; P1.epi = ws;
          if (tc32) set_terms(P1, r);
          if (dw_k_limit) { P1.k_limit = a->row_limit; P1.k_base = lo; }
          rc = tc::launch_tc_gemm(&As1, &Bs1, &P1, 1, gdt, sched + 2 * L.nchunks + 2 + sl, st);
        }
        if (!rc) {
          LK_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(a->grad_w_slice_events[sl]), st));
          recorded = sl + 1;
        }
      }
    } else {
      if (a->grad_x) {
        Operand A{zbuf, L.ldz, 1}, B{a->weight, 1, H};
        rc = launch_simt_gemm(A, B, r, H, V, dt, xe, st);
        if (rc) return rc;
      }
      if (a->grad_w) {
        Operand A{zbuf, 1, L.ldz}, B{xc, 1, H};
        rc = launch_simt_gemm(A, B, V, H, r, dt, we, st);
      }
    }
    if (rc) return rc;
  }
  ProfScope ps_tail(3, st);
  if (want_grad && a->grad_w && dt != LK_F32 && L.nchunks > 1 && !wacc && separate_cast()) {
    rc = launch_cast_f32(dwacc, a->grad_w, V * H, dt, st);
    if (rc) return rc;
  }
  if (a->grad_bias) {
    rc = launch_colsum_rows(bacc, 1, V, V, LK_F32, a->grad_bias, dt, 0, st);
    if (rc) return rc;
  }
  if (a->loss_sum) { rc = launch_reduce_sum(a->loss_rows, BT, a->loss_sum, st); if (rc) return rc; }
  if (a->z_loss_sum && a->z_loss_rows) {
    rc = launch_reduce_sum(a->z_loss_rows, BT, a->z_loss_sum, st);
    if (rc) return rc;
  }
  return record_rest();
}

// ------------------------------------------------------ vocab-parallel ----
extern "C" size_t lk_flce_vp_workspace_bytes(int64_t rows, int64_t hidden, int64_t vocab_local, int dtype) {
  (void)hidden;
  const int64_t nparts = (vocab_local + tc::BN - 1) / tc::BN;
  return align_up((size_t)rows * nparts * sizeof(float4), 1024) + align_up((size_t)rows * 4, 1024) + 4096 +
         (size_t)elt_size(dtype) * 0;
}

// Stage 1: local-shard logits + per-row local statistics (max, sumexp, sum_logits, target_logit).
extern "C" int lk_flce_vp_logits(const void* x, const void* weight_shard, const int64_t* target, int64_t rows,
                                 int64_t hidden, int64_t vocab_local, int64_t vocab_offset, int dtype,
                                 int64_t ignore_index, float softcap, float* row_stats, void* logits_buf,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  LK_REQUIRE(rows >= 0 && hidden >= 1 && vocab_local >= 1, LK_SIZE_MISMATCH, "bad sizes");
  LK_REQUIRE(workspace && workspace_bytes >= lk_flce_vp_workspace_bytes(rows, hidden, vocab_local, dtype),
             LK_INVALID_ARGUMENT, "workspace too small");
  if (rows == 0) return LK_OK;
  cudaStream_t st = as_stream(stream);
  const bool tc = use_tc_path(dtype, hidden, x, weight_shard, 0);
  const int64_t ldz = ld_logits(vocab_local);
  const int64_t nparts = (vocab_local + tc::BN - 1) / tc::BN;
  char* ws = static_cast<char*>(workspace);
  float4* parts = reinterpret_cast<float4*>(ws);
  float* tgt = reinterpret_cast<float*>(ws + align_up((size_t)rows * nparts * sizeof(float4), 1024));
  int* sched = reinterpret_cast<int*>(ws + align_up((size_t)rows * nparts * sizeof(float4), 1024) +
                                      align_up((size_t)rows * 4, 1024));
  EpiArgs le{};
  le.kind = EPI_LOGITS; le.out_dtype = dtype; le.out = logits_buf; le.ldo = ldz; le.alpha = 1.f;
  le.softcap = softcap; le.target = target; le.col_offset = vocab_offset; le.ignore_index = ignore_index;
  le.partials = parts; le.n_parts = nparts; le.tgt_logit = tgt; le.M = rows; le.N = vocab_local;
  le.want_sum = 1;
  int rc;
  LK_CUDA(cudaMemsetAsync(tgt, 0, (size_t)rows * 4, st));
  if (tc) {
    LK_CUDA(cudaMemsetAsync(sched, 0, 64, st));
    tc::TmaOperand A{x, hidden, rows, hidden, 0}, B{weight_shard, hidden, vocab_local, hidden, 0};
    tc::Problem P{};
    P.M = rows; P.N = vocab_local; P.K = hidden; P.n_fast = 0; P.epi = le;
    ProfScope ps(0, st);  // stage timing as in the token-local loop (logits GEMM)
    rc = tc::launch_tc_gemm(&A, &B, &P, 1, dtype, sched, st);
  } else {
    Operand A{x, hidden, 1}, B{weight_shard, hidden, 1};
    rc = launch_simt_gemm(A, B, rows, vocab_local, hidden, dtype, le, st);
  }
  if (rc) return rc;
  // reduce the per-tile partials (tc) or the stored row (simt) to one stats row
  return launch_vp_row_stats(logits_buf, ldz, rows, vocab_local, dtype, target, vocab_offset, ignore_index,
                             tc ? parts : nullptr, nparts, tgt, reinterpret_cast<float4*>(row_stats), st);
}

extern "C" int lk_flce_vp_backward2(const void* x, const void* weight_shard, const int64_t* target, int64_t rows,
                                    int64_t hidden, int64_t vocab_local, int64_t vocab_offset, int64_t vocab_total,
                                    int dtype, int64_t ignore_index, float label_smoothing, float lse_square_scale,
                                    float softcap, int reduction, const int64_t* n_non_ignore,
                                    const float* row_stats_global, void* logits_buf, float* loss_rows,
                                    void* grad_x_partial, int grad_x_dtype, void* grad_w_accum, int grad_w_dtype,
                                    int accumulate, void* workspace, size_t workspace_bytes, void* stream) {
  LK_REQUIRE(rows >= 0 && hidden >= 1 && vocab_local >= 1, LK_SIZE_MISMATCH, "bad sizes");
  LK_REQUIRE(grad_x_dtype == LK_F32 || grad_x_dtype == dtype, LK_INVALID_ARGUMENT,
             "grad_x partial must be fp32 or the input dtype");
  if (rows == 0) return LK_OK;
  cudaStream_t st = as_stream(stream);
  const int64_t ldz = ld_logits(vocab_local);
  CeRowArgs ce{};
  ce.x = logits_buf; ce.ld = ldz; ce.target = target; ce.rows = rows; ce.n_cols = vocab_local;
  ce.vocab_total = vocab_total; ce.col_offset = vocab_offset; ce.ignore_index = ignore_index;
  ce.label_smoothing = label_smoothing; ce.lse_square_scale = lse_square_scale; ce.softcap = softcap;
  ce.input_capped = 1; ce.reduction = reduction; ce.compute_grad = 1; ce.n_valid = n_non_ignore;
  ce.loss_rows = loss_rows; ce.row_stats = reinterpret_cast<const float4*>(row_stats_global);
  int rc;
  {
    ProfScope ps(1, st);  // finalize
    rc = launch_ce_ring(ce, dtype, st);  // persistent TMA ring; the block kernel for other shapes
    if (rc == LK_UNSUPPORTED) rc = launch_ce_rows(ce, dtype, st);
  }
  if (rc) return rc;
  // dX partial (fp32 or the input dtype, all-reduced by the caller) and the local dW shard
  void* grad_x_partial_f32 = grad_x_partial;
  EpiArgs xe{};
  xe.kind = EPI_STORE; xe.out_dtype = grad_x_dtype; xe.out = grad_x_partial; xe.ldo = hidden; xe.alpha = 1.f;
  xe.M = rows; xe.N = hidden;
  EpiArgs we{};
  LK_REQUIRE(grad_w_dtype == LK_F32 || grad_w_dtype == dtype, LK_INVALID_ARGUMENT,
             "grad_w accumulator must be fp32 or the weight dtype");
  we.kind = EPI_ACCUM; we.ldacc = hidden; we.ldo = hidden; we.alpha = 1.f;
  we.beta = accumulate ? 1 : 0; we.M = vocab_local; we.N = hidden;
  if (grad_w_dtype == LK_F32) {  // fp32 accumulator
    we.out_dtype = LK_F32; we.acc = static_cast<float*>(grad_w_accum);
  } else {  // weight-dtype accumulation in place (Liger accum_dtype=None order; TMA reduce-add)
    we.out_dtype = dtype; we.acc = nullptr; we.out = grad_w_accum; we.final_out = 0;
  }
  const bool tc = use_tc_path(dtype, hidden, x, weight_shard, 0) && workspace && workspace_bytes >= 64;
  if (tc) {
    // both GEMMs in one persistent tcgen05 launch, as in the token-local FLCE backward:
    // dX partial (fp32, all-reduced by the caller) = dZ W_shard; dW_shard (+)= dZ^T X (fp32)
    tc::TmaOperand As[2], Bs[2];
    tc::Problem Ps[2];
    int np = 0;
    if (grad_x_partial_f32) {
      if (grad_x_dtype == LK_F32) xe.kind = EPI_F32;  // else EPI_STORE in the input dtype (TMA store)
      As[np] = {logits_buf, vocab_local, rows, ldz, 0};
      Bs[np] = {weight_shard, hidden, vocab_local, hidden, 1};
      Ps[np] = tc::Problem{};
      Ps[np].M = rows; Ps[np].N = hidden; Ps[np].K = vocab_local; Ps[np].n_fast = 0; Ps[np].epi = xe;
      ++np;
    }
    if (grad_w_accum) {
      As[np] = {logits_buf, vocab_local, rows, ldz, 1};
      Bs[np] = {x, hidden, rows, hidden, 1};
      Ps[np] = tc::Problem{};
      Ps[np].M = vocab_local; Ps[np].N = hidden; Ps[np].K = rows; Ps[np].n_fast = 1; Ps[np].epi = we;
      ++np;
    }
    if (!np) return LK_OK;
    int* sched = static_cast<int*>(workspace);
    LK_CUDA(cudaMemsetAsync(sched, 0, 64, st));
    ProfScope ps(2, st);  // backward GEMM (dX partial + dW shard)
    return tc::launch_tc_gemm(As, Bs, Ps, np, dtype, sched, st);
  }
  if (grad_x_partial_f32) {
    Operand A{logits_buf, ldz, 1}, B{weight_shard, 1, hidden};
    rc = launch_simt_gemm(A, B, rows, hidden, vocab_local, dtype, xe, st);
    if (rc) return rc;
  }
  if (grad_w_accum) {
    Operand A{logits_buf, 1, ldz}, B{x, 1, hidden};
    rc = launch_simt_gemm(A, B, vocab_local, hidden, rows, dtype, we, st);
  }
  return rc;
}

extern "C" int lk_flce_vp_backward_ex(const void* x, const void* weight_shard, const int64_t* target, int64_t rows,
                                      int64_t hidden, int64_t vocab_local, int64_t vocab_offset, int64_t vocab_total,
                                      int dtype, int64_t ignore_index, float label_smoothing, float lse_square_scale,
                                      float softcap, int reduction, const int64_t* n_non_ignore,
                                      const float* row_stats_global, void* logits_buf, float* loss_rows,
                                      void* grad_x_partial_f32, void* grad_w_accum, int grad_w_dtype, int accumulate,
                                      void* workspace, size_t workspace_bytes, void* stream) {
  return lk_flce_vp_backward2(x, weight_shard, target, rows, hidden, vocab_local, vocab_offset, vocab_total, dtype,
                              ignore_index, label_smoothing, lse_square_scale, softcap, reduction, n_non_ignore,
                              row_stats_global, logits_buf, loss_rows, grad_x_partial_f32, LK_F32, grad_w_accum,
                              grad_w_dtype, accumulate, workspace, workspace_bytes, stream);
}

extern "C" int lk_flce_vp_backward(const void* x, const void* weight_shard, const int64_t* target, int64_t rows,
                                   int64_t hidden, int64_t vocab_local, int64_t vocab_offset, int64_t vocab_total,
                                   int dtype, int64_t ignore_index, float label_smoothing, float lse_square_scale,
                                   float softcap, int reduction, const int64_t* n_non_ignore,
                                   const float* row_stats_global, void* logits_buf, float* loss_rows,
                                   void* grad_x_partial_f32, float* grad_w_accum, int accumulate, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  return lk_flce_vp_backward_ex(x, weight_shard, target, rows, hidden, vocab_local, vocab_offset, vocab_total, dtype,
                                ignore_index, label_smoothing, lse_square_scale, softcap, reduction, n_non_ignore,
                                row_stats_global, logits_buf, loss_rows, grad_x_partial_f32, grad_w_accum, LK_F32,
                                accumulate, workspace, workspace_bytes, stream);
}

// ------------------------------------------------------------ GEMM test ----
extern "C" int lk_gemm_test(const void* a, const void* b, float* d, int64_t m, int64_t n, int64_t k, int layout,
                            int dtype, int use_tcgen05, void* workspace, size_t workspace_bytes, void* stream) {
  LK_REQUIRE(a && b && d, LK_INVALID_ARGUMENT, "null pointer");
  LK_REQUIRE(layout >= 0 && layout <= 2, LK_INVALID_ARGUMENT, "layout must be 0, 1 or 2");
  cudaStream_t st = as_stream(stream);
  EpiArgs e{};
  e.kind = EPI_F32; e.out_dtype = LK_F32; e.out = d; e.ldo = n; e.M = m; e.N = n; e.alpha = 1.f;
  if (use_tcgen05) {
#ifdef LK_HAS_TCGEN05
    LK_REQUIRE(workspace && workspace_bytes >= 64, LK_INVALID_ARGUMENT, "workspace too small");
    LK_CUDA(cudaMemsetAsync(workspace, 0, 64, st));
    tc::TmaOperand A, B;
    if (layout == 0) { A = {a, k, m, k, 0}; B = {b, k, n, k, 0}; }
    else if (layout == 1) { A = {a, k, m, k, 0}; B = {b, n, k, n, 1}; }
    else { A = {a, m, k, m, 1}; B = {b, n, k, n, 1}; }
    LK_REQUIRE(tc::tma_ok(A) && tc::tma_ok(B), LK_NON_CONTIGUOUS, "operands not TMA-describable");
    tc::Problem P{};
    P.M = m; P.N = n; P.K = k; P.n_fast = layout == 2 ? 1 : 0; P.epi = e;
    return tc::launch_tc_gemm(&A, &B, &P, 1, dtype, static_cast<int*>(workspace), st, use_tcgen05 == 2 ? 2 : 1);
#else
    return fail(LK_UNSUPPORTED, "built without tcgen05");
#endif
  }
  Operand A, B;
  if (layout == 0) { A = {a, k, 1}; B = {b, k, 1}; }
  else if (layout == 1) { A = {a, k, 1}; B = {b, 1, n}; }
  else { A = {a, 1, m}; B = {b, 1, n}; }
  return launch_simt_gemm(A, B, m, n, k, dtype, e, st);
}

extern "C" int lk_gemm_test_accum16(const void* a, const void* b, void* d16, int64_t m, int64_t n, int64_t k,
                                    int dtype, int beta, int use_tma_reduce, void* workspace,
                                    size_t workspace_bytes, void* stream) {
#ifdef LK_HAS_TCGEN05
  LK_REQUIRE(a && b && d16 && workspace && workspace_bytes >= 64, LK_INVALID_ARGUMENT, "null pointer / workspace");
  cudaStream_t st = as_stream(stream);
  LK_CUDA(cudaMemsetAsync(workspace, 0, 64, st));
  EpiArgs e{};
  e.kind = EPI_ACCUM; e.out_dtype = dtype; e.out = d16; e.ldo = n; e.M = m; e.N = n; e.alpha = 1.f;
  e.acc = nullptr; e.ldacc = n; e.beta = beta; e.final_out = 0;
  tc::TmaOperand A{a, k, m, k, 0}, B{b, k, n, k, 0};
  tc::Problem P{};
  P.M = m; P.N = n; P.K = k; P.n_fast = 0; P.epi = e;
  return tc::launch_tc_gemm(&A, &B, &P, 1, dtype, static_cast<int*>(workspace), st, 0, !use_tma_reduce);
#else
  return fail(LK_UNSUPPORTED, "built without tcgen05");
#endif
}
