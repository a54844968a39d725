/*
 * liger_b200.h — C ABI of the B200-native (sm_100a) Liger training hot path.
 *
 * This is the drop-in boundary for the reference's fused-kernel layer
 * (/root/reference/pkg/src/rowfuse/ops.py and flce.py, surveyed in SURVEY.md
 * §8(a)/(b)) and for the third-party Liger operator surface those kernels stand
 * for (liger_kernel 0.8.0, the ops package).  The reference is pure Python, so there is
 * no FFI to replace; each entry point below is what a ctypes/cffi binding of the
 * reference's operator would call (see INTEGRATION.md for the binding stubs).
 *
 * Conventions (all entry points):
 *   - Plain device pointers, int64 sizes, a cudaStream_t passed as void*.
 *   - The library never allocates device memory: scratch is a caller-provided
 *     workspace sized by the matching *_workspace_bytes() query.  Peak memory is
 *     therefore attributable to the caller's allocator (SURVEY §8(b) ownership).
 *   - Calls are stream-ordered and asynchronous; none of them synchronises the
 *     host.  Target-range violations are reported through a device flag written
 *     into the workspace (lk_status LK_TARGET_OUT_OF_RANGE is set by the host
 *     wrapper after reading it), mirroring rowfuse's TargetOutOfRange
 *     (rowfuse/core.py:45-46, ops.py:489-499).
 *   - Return value: 0 on success, otherwise an lk_status code; the message is
 *     available from lk_last_error() (thread-local).  Status codes mirror the
 *     reference error taxonomy (rowfuse/core.py:25-46).
 *   - All offsets are computed in 64-bit (rowfuse/core.py:86-94 makes 64-bit
 *     offsets a design decision once rows*cols-1 > 2^31-1; cfg4/cfg5 exceed it).
 */
#ifndef LIGER_B200_H
#define LIGER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- types ------------------------------------------------------------- */

typedef enum {
  LK_F32 = 0,
  LK_BF16 = 1,
  LK_F16 = 2
} lk_dtype;

typedef enum {
  LK_OK = 0,
  LK_NON_CONTIGUOUS = 1,      /* rowfuse/core.py:33-39 NonContiguousInput   */
  LK_SHAPE_MISMATCH = 2,      /* rowfuse/core.py:29-30 ShapeMismatch        */
  LK_SIZE_MISMATCH = 3,       /* rowfuse/core.py:25-26 SizeMismatch         */
  LK_ODD_HEAD_DIM = 4,        /* rowfuse/core.py:41-42 OddHeadDim           */
  LK_TARGET_OUT_OF_RANGE = 5, /* rowfuse/core.py:45-46 TargetOutOfRange     */
  LK_UNSUPPORTED = 6,         /* option the kernels do not implement         */
  LK_CUDA_ERROR = 7,          /* launch / runtime failure                     */
  LK_INVALID_ARGUMENT = 8     /* null pointer, bad enum, workspace too small  */
} lk_status;

typedef enum {
  LK_REDUCTION_NONE = 0,
  LK_REDUCTION_MEAN = 1, /* Liger: mean over non-ignored rows (LK/ops/cross_entropy.py:218-219) */
  LK_REDUCTION_SUM = 2
} lk_reduction;

typedef enum {
  LK_CAST_LLAMA = 0, /* LK/ops/rms_norm.py:83-112: rstd fp32, xhat cast before *w */
  LK_CAST_GEMMA = 1, /* all fp32, cast at the end                                */
  LK_CAST_NONE = 2   /* compute in the input dtype                              */
} lk_casting_mode;

/* ---- library ----------------------------------------------------------- */

const char* lk_last_error(void);
const char* lk_version(void);
/* 1 if the .so was built with the sm_100a tcgen05 GEMM path. */
int lk_has_tcgen05(void);

/* Instrumentation for the benchmark (off by default).  When enabled, the FLCE
 * entry points record CUDA events on the launching stream around each stage:
 *   0 = logits GEMM (tcgen05 or SIMT), 1 = finalize (softmax-grad rows),
 *   2 = backward GEMM (dX + dW), 3 = other (target count, loss reduction, bias).
 * lk_profile_collect() waits for the recorded events, writes the summed
 * milliseconds and launch counts per stage, and clears the record.
 * lk_launch_count() is the number of kernels this library has launched. */
void lk_profile_enable(int on);
int lk_profile_collect(double* ms4, int64_t* launches4);
int64_t lk_launch_count(void);

/* TEST-ONLY path selection.  The library runs one product path per shape; the kernels it
 * replaced stay selectable here so the parity tests can run each against the others.  Knobs
 * are process-wide and default to 0 = the product path; nothing reads the environment.
 *   LK_PATH_CTA_GROUP          0 = CTA-pair tcgen05 GEMM, 1 = single-CTA GEMM
 *   LK_PATH_FLCE_FINALIZE      0 = TMA-ring finalize, 1 = one CTA per row (ce_rows_kernel)
 *   LK_PATH_FLCE_SEPARATE_CAST 0 = fp32 dW accumulator folded into the last chunk's epilogue,
 *                              1 = separate cast kernel after the loop
 *   LK_PATH_CE_IMPL            0 = TMA-ring CE, 1 = one CTA per row
 *   LK_PATH_NORM_IMPL          0 = CTA-per-row RMSNorm, 1 = warp per row, 2 = generic, 3 = TMA ring
 *   LK_PATH_DW_ACCUM16         0 = 16-bit grad_w accumulation by TMA reduce-add in L2,
 *                              1 = read-add-round in the epilogue registers
 * Returns the previous value, or -1 for an unknown knob / value. */
#define LK_PATH_CTA_GROUP 0
#define LK_PATH_FLCE_FINALIZE 1
#define LK_PATH_FLCE_SEPARATE_CAST 2
#define LK_PATH_CE_IMPL 3
#define LK_PATH_NORM_IMPL 4
#define LK_PATH_DW_ACCUM16 5
int lk_test_select_path(int knob, int value);

/* ---- cross entropy (standalone) ---------------------------------------- */
/*
 * Replaces rowfuse.ops.cross_entropy (rowfuse/ops.py:502-560) and
 * liger_kernel.ops.cross_entropy.cross_entropy_forward (LK/ops/cross_entropy.py:302-407).
 * logits[rows, ld] (row-major, unit column stride) is overwritten in place with
 * d(loss)/d(logits) when compute_grad != 0.  loss_rows[rows] (fp32) receives the
 * per-row loss (already divided by the non-ignored count for MEAN);
 * loss_sum (fp32 scalar, may be NULL) receives the deterministic sum of loss_rows.
 * z_loss_rows / z_loss_sum optional (lse_square_scale term).
 * softcap <= 0 means "no softcap".
 */
size_t lk_cross_entropy_workspace_bytes(int64_t rows);
int lk_cross_entropy_fwd(void* logits, int64_t ld, const int64_t* targets, int64_t rows,
                         int64_t vocab, int dtype, int64_t ignore_index, float label_smoothing,
                         float lse_square_scale, float softcap, int reduction, int compute_grad,
                         float* loss_rows, float* loss_sum, float* z_loss_rows, float* z_loss_sum,
                         void* workspace, size_t workspace_bytes, void* stream);
/* Same, plus Liger's return_token_accuracy / return_predicted_tokens outputs: per row
 * 1.0 if argmax == target else 0.0 (correct_rows) and the argmax (pred_rows); ignored rows
 * -> 0.0 / -1; either may be NULL (LK/ops/cross_entropy.py:131-163, 294-299).  class_weight
 * ([vocab] fp32 or NULL) is Liger's `weight` (LK/ops/cross_entropy.py:122-124, 220-239,
 * 278-288), also combined with label_smoothing (the smoothing term weighted as Liger does). */
int lk_cross_entropy_fwd_ex(void* logits, int64_t ld, const int64_t* targets, int64_t rows, int64_t vocab,
                            int dtype, int64_t ignore_index, float label_smoothing, float lse_square_scale,
                            float softcap, int reduction, int compute_grad, float* loss_rows, float* loss_sum,
                            float* z_loss_rows, float* z_loss_sum, float* correct_rows, int64_t* pred_rows,
                            const float* class_weight, void* workspace, size_t workspace_bytes, void* stream);

/* Count of targets != ignore_index and the out-of-range flag, on device.
 * out[0] = n_non_ignore (as int64), out[1] = number of out-of-range targets. */
int lk_count_targets(const int64_t* targets, int64_t rows, int64_t vocab, int64_t ignore_index,
                     int64_t* out, void* stream);

/* x[rows, cols] (row stride ld) *= scale, where scale is a device fp32 scalar
 * (grad_output of a reduced loss) — the backward of CE/FLCE
 * (LK/ops/cross_entropy.py:415-440, LK/ops/fused_linear_cross_entropy.py:247-291).
 * The kernel early-exits when *scale == 1.0f, so no host sync is needed.  */
int lk_scale_by_device_scalar(void* x, int64_t rows, int64_t cols, int64_t ld, int dtype,
                              const float* scale, void* stream);
/* x[r, :] *= row_scale[r] (reduction="none" backward, LK/ops/cross_entropy.py:424-426). */
int lk_scale_rows(void* x, int64_t rows, int64_t cols, int64_t ld, int dtype,
                  const void* row_scale, int row_scale_dtype, void* stream);

/* ---- fused linear cross entropy ---------------------------------------- */
/*
 * Replaces rowfuse.flce.flce_forward_backward (rowfuse/flce.py:107-173) and
 * liger_kernel's fused_linear_cross_entropy_forward (LK/ops/fused_linear_cross_entropy.py:17-244).
 * Layout follows Liger: x[BT, H], weight[V, H] (rowfuse stores W as (H, V); the
 * Python adapter transposes for the oracle).  Gradients are produced during the
 * forward: grad_x[BT, H] in x's dtype, grad_w[V, H] in weight's dtype (accumulated
 * across chunks per grad_w_accum below).  Either grad pointer may be NULL to
 * skip that gradient.  chunk_rows <= 0 selects the B200 chunk policy
 * (lk_flce_plan); otherwise any positive row count is honoured (the reference's
 * ChunkPlan.with_chunk_rows override, rowfuse/flce.py:58-66).
 */
typedef struct {
  const void* x;          /* [BT, H] contiguous                                */
  const void* weight;     /* [V, H] contiguous                                 */
  const int64_t* target;  /* [BT]                                              */
  const void* bias;       /* [V] or NULL                                       */
  int64_t bt, hidden, vocab;
  int dtype;              /* lk_dtype of x and weight (must match)             */
  int64_t ignore_index;
  float label_smoothing;
  float lse_square_scale;
  float softcap;          /* <= 0: none                                        */
  int reduction;          /* lk_reduction                                      */
  int64_t chunk_rows;     /* <= 0: lk_flce_plan                                */
  /* outputs */
  float* loss_rows;       /* [BT] fp32 (required)                              */
  float* loss_sum;        /* scalar fp32 or NULL                               */
  float* z_loss_rows;     /* [BT] fp32 or NULL                                 */
  float* z_loss_sum;      /* scalar or NULL                                    */
  void* grad_x;           /* [BT, H] dtype or NULL                             */
  void* grad_w;           /* [V, H] dtype or NULL                              */
  void* grad_bias;        /* [V] dtype or NULL                                 */
  int64_t* target_stats;  /* [2] n_non_ignore, n_out_of_range (device) or NULL */
  /* scratch */
  void* workspace;
  size_t workspace_bytes;
  void* stream;
  int force_simt;         /* 1: the SIMT FFMA GEMMs (test reference for fp32)   */
  /* Token-sharded mode: device int64 holding the GLOBAL non-ignored count used as
   * the MEAN denominator (all-reduced by the caller); NULL = local count. */
  const int64_t* mean_count;
  /* grad_w accumulation across chunks (Liger's accum_dtype,
   * LK/ops/fused_linear_cross_entropy.py:64-69): LK_ACCUM_AUTO (0, the zero-initialised
   * default) = weight dtype when the plan has <= LK_ACCUM_AUTO_MAX_CHUNKS chunks (a bf16
   * TMA reduce-add in L2, no fp32 workspace, peak memory ~ one logits chunk), else fp32;
   * LK_ACCUM_FP32 = fp32 workspace accumulator; LK_ACCUM_WEIGHT_DTYPE = always the weight
   * dtype (Liger's accum_dtype=None semantics). */
  int grad_w_accum;
  /* Liger return_token_accuracy / return_predicted_tokens (LK/ops/fused_linear_cross_entropy.py:
   * 119-125, 148-160): per row 1.0 if argmax(logits) == target else 0.0, and the argmax
   * (first column of the max of the softcapped, rounded logits); ignored rows -> 0.0 / -1.
   * NULL = not computed (the epilogue then skips the argmax search). */
  float* token_correct_rows;  /* [BT] fp32 or NULL */
  int64_t* predicted_tokens;  /* [BT] or NULL      */
  /* Token-sharded overlap: grad_w_slice_events[0 .. grad_w_slices) are
   * cudaEvents created by the caller; slice s = grad_w rows [s*R, min(V, (s+1)*R)) with
   * R = round_up(ceil(V/S), 256).  Contract: event s is recorded on `stream` after slice s of
   * grad_w is final, on EVERY successful path.  On the tcgen05 path with
   * 2 <= S <= LK_MAX_GRAD_W_SLICES the last chunk's grad_w GEMM runs as S launches and event s
   * follows launch s (so the caller all-reduces slice s while later slices compute); on any
   * other path (SIMT/fp32, BT == 0, other S) every event is recorded after all of grad_w. */
  int grad_w_slices;
  void* const* grad_w_slice_events;
  /* Liger use_token_scaling (LK/ops/fused_linear_cross_entropy.py:109-139, 187-206): each
   * row's loss, z-loss and gradient scaled by its detached target probability. */
  int use_token_scaling;
  /* Liger ce_weight: [vocab] fp32 class weights or NULL. */
  const float* ce_weight;
  /* Token-sharded mode with ce_weight: device fp32 holding the GLOBAL sum of the valid
   * targets' weights (the weighted MEAN denominator, all-reduced by the caller); NULL =
   * local sum. */
  const float* mean_weight_sum;
  /* fp32 inputs (dtype LK_F32): the GEMMs run on the bf16 tensor cores on operands split
   * into this many bf16 pieces (csrc/split.cu): 3 (default when 0) = 6 piece products per
   * product (products exact to fp32's 2^-24), 2 = 3 products (~2^-16 per product: faster,
   * below the fp32 tolerance on long training runs).  The long-K dX GEMM accumulates in
   * segments added in fp32 (the tensor core's own accumulator truncates).  Ignored for
   * 16-bit dtypes and with force_simt. */
  int fp32_pieces;
  /* Kept-row gather (the ignored-row skipping of fused_linear_cross_entropy.py): NULL, or
   * x_row_index[bt] = the x row of each of the call's bt rows (lk_compact_rows' list).  The
   * chunk loop then gathers each chunk's X rows into a chunk-sized workspace buffer
   * (lk_gather_rows) instead of reading x[lo : lo + r]; everything else -- targets, grad_x,
   * the per-row outputs -- is indexed by the call's rows.  x may hold more rows than bt. */
  const int64_t* x_row_index;
  /* Device-side row count (with x_row_index: the kept-row FLCE without a host read of the
   * count, e.g. under CUDA graph capture): NULL, or a device int64 n <= bt.  The caller
   * guarantees that rows >= n are ignore_index rows whose X rows are zero (x_row_index = -1).
   * The CTA-pair GEMMs then skip the M tiles past row n of each chunk and stop the dW K loop at
   * row max(n, 1).  The outputs are unchanged: a limit only removes work. */
  const int64_t* row_limit;
} lk_flce_args;

/* Workspace bytes for exactly this call (every field that sizes the workspace is read:
 * bt, hidden, vocab, dtype, chunk_rows, grad_w, grad_bias, grad_w_accum, force_simt,
 * fp32_pieces, x_row_index; other pointers may be NULL). */
size_t lk_flce_workspace_bytes_for(const lk_flce_args* args);

enum { LK_ACCUM_AUTO = 0, LK_ACCUM_FP32 = 1, LK_ACCUM_WEIGHT_DTYPE = 2 };
#define LK_ACCUM_AUTO_MAX_CHUNKS 8
#define LK_MAX_GRAD_W_SLICES 16

/* B200 chunk policy.  Writes the chunk row count and number of chunks. */
int lk_flce_plan(int64_t bt, int64_t hidden, int64_t vocab, int dtype, int64_t* chunk_rows,
                 int64_t* num_chunks);
size_t lk_flce_workspace_bytes(int64_t bt, int64_t hidden, int64_t vocab, int dtype,
                               int64_t chunk_rows, int has_grad_w);
/* Same, for an explicit grad_w_accum mode (lk_flce_workspace_bytes assumes LK_ACCUM_AUTO). */
size_t lk_flce_workspace_bytes_ex(int64_t bt, int64_t hidden, int64_t vocab, int dtype,
                                  int64_t chunk_rows, int has_grad_w, int grad_w_accum);
int lk_flce_forward_backward(const lk_flce_args* args);

/*
 * Staged FLCE entry points for the vocab-parallel mode: each rank
 * holds weight rows [v0, v0+vocab_local).  Stage 1 produces per-row partial
 * softmax statistics for the local shard; the caller all-reduces them across
 * ranks (max, then rescaled sum), then stage 2 writes dlogits for the local
 * shard and accumulates grad_x (to be all-reduced by the caller) and the local
 * grad_w shard.
 *   row_stats layout: [rows, 4] fp32 = (max, sumexp, sum_logits, target_logit),
 *   target_logit is 0 on ranks that do not own the target column.
 */
size_t lk_flce_vp_workspace_bytes(int64_t rows, int64_t hidden, int64_t vocab_local, int dtype);
int lk_flce_vp_logits(const void* x, const void* weight_shard, const int64_t* target, int64_t rows,
                      int64_t hidden, int64_t vocab_local, int64_t vocab_offset, int dtype,
                      int64_t ignore_index, float softcap, float* row_stats, void* logits_buf,
                      void* workspace, size_t workspace_bytes, void* stream);
int lk_flce_vp_backward(const void* x, const void* weight_shard, const int64_t* target,
                        int64_t rows, int64_t hidden, int64_t vocab_local, int64_t vocab_offset,
                        int64_t vocab_total, int dtype, int64_t ignore_index, float label_smoothing,
                        float lse_square_scale, float softcap, int reduction,
                        const int64_t* n_non_ignore, const float* row_stats_global,
                        void* logits_buf, float* loss_rows, void* grad_x_partial_f32,
                        float* grad_w_accum, int accumulate, void* workspace,
                        size_t workspace_bytes, void* stream);
/* As lk_flce_vp_backward, with the dW shard accumulated either in fp32 (grad_w_dtype = LK_F32)
 * or in place in the weight dtype (grad_w_dtype = dtype: dtype(acc + dtype(chunk product)),
 * Liger's accum_dtype=None order, as lk_flce_args.grad_w_accum = LK_ACCUM_WEIGHT_DTYPE). */
int lk_flce_vp_backward_ex(const void* x, const void* weight_shard, const int64_t* target, int64_t rows,
                           int64_t hidden, int64_t vocab_local, int64_t vocab_offset, int64_t vocab_total, int dtype,
                           int64_t ignore_index, float label_smoothing, float lse_square_scale, float softcap,
                           int reduction, const int64_t* n_non_ignore, const float* row_stats_global,
                           void* logits_buf, float* loss_rows, void* grad_x_partial_f32, void* grad_w_accum,
                           int grad_w_dtype, int accumulate, void* workspace, size_t workspace_bytes, void* stream);

/* As lk_flce_vp_backward_ex with the dX partial written in grad_x_dtype (LK_F32, or the input
 * dtype so the caller all-reduces it in place in 16-bit: half the bytes of the fp32 partial). */
int lk_flce_vp_backward2(const void* x, const void* weight_shard, const int64_t* target, int64_t rows,
                         int64_t hidden, int64_t vocab_local, int64_t vocab_offset, int64_t vocab_total, int dtype,
                         int64_t ignore_index, float label_smoothing, float lse_square_scale, float softcap,
                         int reduction, const int64_t* n_non_ignore, const float* row_stats_global,
                         void* logits_buf, float* loss_rows, void* grad_x_partial, int grad_x_dtype,
                         void* grad_w_accum, int grad_w_dtype, int accumulate, void* workspace,
                         size_t workspace_bytes, void* stream);
/* Combine the all-gathered per-rank row statistics gathered[world][rows][4] into the global
 * row_stats[rows][4] (max; sumexp rescaled to the global max; sums), folding ranks in rank
 * order so every rank gets bit-identical statistics. */
int lk_flce_vp_combine_stats(const float* gathered, int64_t world, int64_t rows, float* row_stats, void* stream);

/* ---- ignored-row compaction (fused_linear_cross_entropy.py) ------------------ */
/* Rows whose target is ignore_index contribute nothing to the FLCE (loss 0, gradient row 0, no
 * dW / db term: rowfuse/ops.py:515-523, rowfuse/flce.py:161-168), so the host wrapper runs the
 * chunk loop on the other rows only.  lk_compact_rows writes the stable list of kept rows
 * index[0 .. *count) (index[i] = -1 past the count) and the inverse map pos[rows] (-1 for an
 * ignored row); *count is on the device.  lk_gather_rows copies dst[i, :] = src[index[i], :]
 * for i < out_rows, or the fill element (elem_bytes wide, low bytes of `fill`) where
 * index[i] < 0: with `index` the gather, with `pos` the scatter back. */
int lk_compact_rows(const int64_t* targets, int64_t rows, int64_t ignore_index, int64_t* index, int64_t* pos,
                    int64_t* count, void* stream);
int lk_gather_rows(const void* src, int64_t cols, int elem_bytes, const int64_t* index, int64_t out_rows, void* dst,
                   uint64_t fill, void* stream);

/* ---- peer-memory grad_w all-reduce -------------------- */
/* The token-sharded dW reduction over NVLink peer memory, replacing the NCCL all-reduce of
 * distributed.py (the reference's contract: dW is additive over row shards,
 * /root/reference/pkg/tests/test_flce.py:182-205).  Every rank allocates one symmetric buffer
 * (a control page of LK_PEER_CTL_BYTES, then the data) and maps every peer's buffer through
 * CUDA IPC.  lk_peer_alloc is the one entry point that allocates device memory: IPC needs a
 * cudaMalloc base.  Buffers start zeroed (the control page must be). */
#define LK_PEER_MAX 16
#define LK_PEER_CTL_BYTES 4096
#define LK_PEER_HANDLE_BYTES 64
int lk_peer_alloc(int device, size_t data_bytes, void** base, void* ipc_handle);
/* Maps a peer's buffer from its handle (not the caller's own: use its base directly). */
int lk_peer_open(int device, const void* ipc_handle, void** base);
int lk_peer_close(int device, void* peer_base);
int lk_peer_free(int device, void* base);
/* In-place sum over ranks of n elements (dtype) at byte offset `offset` (from each base; a
 * multiple of the element size) of every rank's buffer.  One kernel: rank r owns the r-th
 * 16-byte-aligned part of the range, loads it from every peer, adds in fp32 in rank order
 * (bit-identical on every rank and every run), rounds once, and stores the sum into every
 * peer.  Flags in the control pages order it: a rank's part is read only after that rank
 * signalled `epoch` (its data final, stream order), and the kernel ends only after every owner
 * signalled its stores done.  Every rank must issue the same calls in the same order with
 * epochs 1, 2, 3, ... per buffer, on one stream per buffer.  A wait longer than timeout_ns
 * (0 = 120 s) abandons the call and sets the buffer's error flag (lk_peer_status) instead of
 * hanging the GPU. */
int lk_peer_allreduce(void* const* bases, int world, int rank, int64_t offset, int64_t n, int dtype,
                      uint64_t epoch, int64_t timeout_ns, void* stream);
/* Synchronous read of the caller's own buffer error flag (1 = a call timed out); clear != 0
 * resets it. */
int lk_peer_status(int device, void* base, int clear, int* error);

/* ---- RMSNorm ----------------------------------------------------------- */
/* rowfuse/ops.py:190-241 and LK/ops/rms_norm.py (forward 58-112, backward 115-210).
 * rstd[rows] is fp32 for llama/gemma casting, x dtype for "none". weight may be NULL
 * (elementwise_affine=False).  dw_partial is a caller workspace of
 * lk_rmsnorm_bwd_workspace_bytes(); dw receives sum over rows in weight dtype. */
int lk_rmsnorm_fwd(const void* x, const void* weight, void* y, void* rstd, int64_t rows,
                   int64_t cols, float eps, float offset, int casting_mode, int dtype, void* stream);
size_t lk_rmsnorm_bwd_workspace_bytes(int64_t rows, int64_t cols);
int lk_rmsnorm_bwd(const void* dy, const void* x, const void* weight, const void* rstd, void* dx,
                   void* dw, int64_t rows, int64_t cols, float offset, int casting_mode, int dtype,
                   void* workspace, size_t workspace_bytes, void* stream);

/* ---- LayerNorm ------------------------------------------ */
/* rowfuse/ops.py:248-311 and LK/ops/layer_norm.py (forward 169-227, backward 230-304).
 * y = (x - mean) * rstd * w + b with rstd = 1/sqrt(mean((x - mean)^2) + eps); mean[rows]
 * and rstd[rows] are fp32.  bias may be NULL (no shift; db then not computed).  cols must be
 * a multiple of 16 bytes.  dw/db are sums over rows in the weight dtype (deterministic two-
 * stage reduction through the caller workspace of lk_layernorm_bwd_workspace_bytes()). */
int lk_layernorm_fwd(const void* x, const void* weight, const void* bias, void* y, float* mean, float* rstd,
                     int64_t rows, int64_t cols, float eps, int dtype, void* stream);
size_t lk_layernorm_bwd_workspace_bytes(int64_t rows, int64_t cols);
int lk_layernorm_bwd(const void* dy, const void* x, const void* weight, const float* mean, const float* rstd,
                     void* dx, void* dw, void* db, int64_t rows, int64_t cols, int dtype, void* workspace,
                     size_t workspace_bytes, void* stream);

/* ---- RoPE -------------------------------------------------------------- */
/* rowfuse/ops.py:344-382 and LK/ops/rope.py:6-112.  q[B, T, nq, d] and
 * k[B, T, nk, d] are rotated in place (half-split HF layout); cos/sin are
 * [cos_batch, T, d] with cos_batch in {1, B}; only cos[..., :d/2] is read.
 * backward != 0 applies the transpose rotation (sin negated). */
int lk_rope(void* q, void* k, const void* cos, const void* sin, int64_t batch, int64_t seq,
            int64_t n_q_heads, int64_t n_kv_heads, int64_t head_dim, int64_t cos_batch,
            int dtype, int cos_dtype, int backward, void* stream);

/* ---- SwiGLU / GeGLU ---------------------------------------------------- */
/* rowfuse/ops.py:389-482, LK/ops/swiglu.py:15-62, LK/ops/geglu.py:23-88.
 * c = act(a) * b over n contiguous elements; backward writes da into a and db
 * into b in place (Liger semantics). */
int lk_swiglu_fwd(const void* a, const void* b, void* c, int64_t n, int dtype, void* stream);
int lk_swiglu_bwd(const void* dc, void* a, void* b, int64_t n, int dtype, void* stream);
int lk_geglu_fwd(const void* a, const void* b, void* c, int64_t n, int dtype, void* stream);
int lk_geglu_bwd(const void* dc, void* a, void* b, int64_t n, int dtype, void* stream);
/* Liger LigerSiLUMulFunction(a, b, gate_multiplier) (LK/ops/swiglu.py:16-62, 113-160):
 * c = silu(gate_multiplier * a) * b; backward da = dc * silu'(gm * a) * b * gm, db = dc * silu(gm * a),
 * written in place.  gate_multiplier == 1 is lk_swiglu_fwd / lk_swiglu_bwd. */
int lk_swiglu_fwd_ex(const void* a, const void* b, void* c, int64_t n, float gate_multiplier, int dtype, void* stream);
int lk_swiglu_bwd_ex(const void* dc, void* a, void* b, int64_t n, float gate_multiplier, int dtype, void* stream);

/* ---- GEMM test hook ----------------------------------------------------- */
/* D[M, N] (fp32, row-major) = A · B for the three operand layouts FLCE uses
 * (layout 0: A[M,K] K-major, B[N,K] K-major; 1: A[M,K] K-major, B[K,N] N-major;
 * 2: A[K,M] M-major, B[K,N] N-major).  use_tcgen05 selects the sm_100a path.
 * Used by the kernel tests only. */
int lk_gemm_test(const void* a, const void* b, float* d, int64_t m, int64_t n, int64_t k,
                 int layout, int dtype, int use_tcgen05, void* workspace, size_t workspace_bytes,
                 void* stream);
/* Test hook for the 16-bit accumulate epilogue: d16[m, n] (weight dtype) = A.B^T
 * (beta = 0, TMA store) or d16 += A.B^T (beta = 1, TMA reduce-add in L2; reduce = 0
 * selects the register read-add-round path), K-major operands, tcgen05. */
int lk_gemm_test_accum16(const void* a, const void* b, void* d16, int64_t m, int64_t n, int64_t k, int dtype,
                         int beta, int use_tma_reduce, void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LIGER_B200_H */
