"""Fused linear cross entropy: LigerFusedLinearCrossEntropyFunction / ...Loss.

Drop-in for liger_kernel's FLCE (LK/transformers/fused_linear_cross_entropy.py:9-69,
LK/ops/fused_linear_cross_entropy.py:17-400).  The algorithm is the reference's
chunked projection head (rowfuse/flce.py:107-173): logits are produced one row
chunk at a time, turned into logit gradients in place, and folded into dX and
dW, so the full BT x V logits never exist.  Everything on the path runs in the
sm_100a library through one C-ABI call (lk_flce_forward_backward); the gradients
are computed during the forward and backward only scales them by grad_output.
"""

from __future__ import annotations

from typing import Optional

import torch

from . import _capi, errors
from ._utils import (
    as_targets,
    check,
    device_guard,
    dtype_code,
    lib,
    ptr,
    count_and_stage_targets,
    raise_if_staged_out_of_range,
    require_contiguous,
    require_cuda,
    stream_of,
    workspace,
)
from .cross_entropy import CrossEntropyOutput


def flce_plan(bt: int, hidden: int, vocab: int, dtype: torch.dtype = torch.bfloat16) -> tuple[int, int]:
    """B200 chunk policy (chunk_rows, num_chunks) from the library (see flce.cu b200_chunk_rows)."""
    c = _capi.C.c_int64()
    n = _capi.C.c_int64()
    code = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}[dtype]
    check(lib().lk_flce_plan(bt, hidden, vocab, code, _capi.C.byref(c), _capi.C.byref(n)))
    return int(c.value), int(n.value)


def flce_workspace_bytes(bt, hidden, vocab, dtype=torch.bfloat16, chunk_rows=None, has_grad_w=True,
                         accum=0) -> int:
    code = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}[dtype]
    return int(lib().lk_flce_workspace_bytes_ex(bt, hidden, vocab, code, int(chunk_rows or 0), int(has_grad_w),
                                                int(accum)))


# Ignored-row skipping (lk_compact_rows / lk_gather_rows, csrc/compact.cu).  On by default for
# calls of at least COMPACT_MIN_SKIPPED rows.  With the host count (KEPT_ROWS_DEVICE_COUNT =
# False) a call skips rows only when at least COMPACT_MIN_SKIPPED rows (and 1/64 of the batch)
# are ignored -- below that the GEMM tiles (256 rows per CTA pair) barely shrink.
SKIP_IGNORED_ROWS = True
COMPACT_MIN_SKIPPED = 128
# Kept-row count without a host read: the FLCE runs on all bt row slots, the kept rows first,
# and the CTA-pair GEMMs read the count on the device (lk_flce_args.row_limit) to skip the M
# tiles and dW K blocks past it -- no host synchronisation anywhere on the call.  Always used
# under CUDA graph capture.  False: the count is read on the host (the chunk plan is then
# sized for the kept rows, and nothing runs when too few rows are ignored); measured equal
# speed at cfg2 (profiles/r02/kept_count_probe*.log).
KEPT_ROWS_DEVICE_COUNT = True


def _gather_rows(src: torch.Tensor, index: torch.Tensor, out_rows: int, dst: torch.Tensor, fill_bits: int = 0):
    cols = src[0].numel() if src.dim() > 1 else 1
    check(lib().lk_gather_rows(src.data_ptr(), cols, src.element_size(), index.data_ptr(), out_rows, dst.data_ptr(),
                               fill_bits, stream_of(src)))
    return dst


class KeptRows:
    """A compaction of one target vector enqueued ahead of the FLCE call that consumes it
    (`prepare_kept_rows`): the kept-row list, the inverse map, and the kept count copied to
    pinned host memory behind an event."""

    def __init__(self, target, index, pos, count, count_host, event):
        # the target tensor itself is held: while the entry exists no other tensor can occupy
        # its memory, so (data pointer, version) identifies it
        self.target, self.index, self.pos, self.count = target, index, pos, count
        self.count_host, self.event = count_host, event
        self.rows = target.numel()

    @property
    def n(self) -> int:
        self.event.synchronize()  # done long ago when prepared early: no wait
        return int(self.count_host[0])


_PREPARED: dict = {}  # (data_ptr, numel, ignore_index, device) -> (version, KeptRows)
_PREPARED_MAX = 8


def _compact(t: torch.Tensor, ignore_index: int):
    bt = t.numel()
    dev = t.device
    index = torch.empty(bt, dtype=torch.int64, device=dev)
    pos = torch.empty(bt, dtype=torch.int64, device=dev)
    count = torch.empty(1, dtype=torch.int64, device=dev)
    check(lib().lk_compact_rows(t.data_ptr(), bt, int(ignore_index), index.data_ptr(), pos.data_ptr(),
                                count.data_ptr(), stream_of(t)))
    return index, pos, count


def prepare_kept_rows(target: torch.Tensor, ignore_index: int = -100,
                      stream: Optional[torch.cuda.Stream] = None) -> Optional[KeptRows]:
    """Enqueue the kept-row compaction of `target` now (e.g. as soon as the labels exist, before
    the model's forward), on `stream` (default: the current stream; the target's producer
    must be ordered before it).  A later FLCE call on the same, unmodified target tensor (same
    storage, same version) then sizes its chunk loop from a count the GPU produced long
    before, instead of waiting for all work queued ahead of it.  That call waits on the
    compaction's event before enqueuing anything that reads its output (host count: on the
    host; device count, the default: on its stream), so `stream` need not be ordered with the
    call's stream, and the call skips its own compaction."""
    t = as_targets(target)
    if not t.is_cuda or t.numel() < COMPACT_MIN_SKIPPED or torch.cuda.is_current_stream_capturing():
        return None
    with torch.cuda.stream(stream or torch.cuda.current_stream(t.device)):
        index, pos, count = _compact(t, ignore_index)
        host = torch.empty(1, dtype=torch.int64, pin_memory=True)
        host.copy_(count, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
    kr = KeptRows(t, index, pos, count, host, ev)
    while len(_PREPARED) >= _PREPARED_MAX:
        _PREPARED.pop(next(iter(_PREPARED)))
    _PREPARED[(t.data_ptr(), t.numel(), int(ignore_index), t.device)] = (t._version, kr)
    return kr


def _take_prepared(t: torch.Tensor, ignore_index: int) -> Optional[KeptRows]:
    """The prepare_kept_rows entry for this exact target tensor (consumed), or None."""
    entry = _PREPARED.pop((t.data_ptr(), t.numel(), int(ignore_index), t.device), None)
    if entry is None or entry[0] != t._version or entry[1].rows != t.numel() \
            or entry[1].target.data_ptr() != t.data_ptr():
        return None
    kr = entry[1]
    cur = torch.cuda.current_stream(t.device)
    for buf in (kr.index, kr.pos, kr.count):  # made on the preparing stream, read on this one
        buf.record_stream(cur)
    return kr


def kept_rows(t: torch.Tensor, ignore_index: int):
    """(index, pos, n) for the rows whose target is not ignore_index: the stable list of kept
    rows, the inverse map (-1 for ignored rows) and their count (lk_compact_rows), or None
    when skipping does not pay (fewer than COMPACT_MIN_SKIPPED or 1/64 of the rows ignored,
    nothing kept) or cannot run (graph capture: the count is a host read).  Uses the
    compaction `prepare_kept_rows` enqueued for this tensor, if any."""
    bt = t.numel()
    if bt < COMPACT_MIN_SKIPPED or torch.cuda.is_current_stream_capturing():
        return None
    kr = _take_prepared(t, ignore_index)
    if kr is not None:
        index, pos, n = kr.index, kr.pos, kr.n
    else:
        index, pos, count = _compact(t, ignore_index)
        n = int(count.item())  # the host read: the chunk loop is sized by the kept rows
    if n == 0 or bt - n < max(COMPACT_MIN_SKIPPED, bt // 64):
        return None
    return index, pos, n


def _forward_kept_rows(x, w, t, ignore_index, need_gx, need_gw, reduction, return_z_loss, return_token_accuracy,
                       return_predicted_tokens, kw):
    """The FLCE on the rows whose target is not ignore_index, outputs scattered back to all rows.

    Ignored rows contribute nothing (loss 0, gradient row 0, no dW / db term:
    rowfuse/ops.py:515-523, rowfuse/flce.py:161-168) and the MEAN denominator counts the kept
    rows only, so the kept-row problem has the same loss, dW and db, and the same dX rows.
    The dW sum is grouped into chunks differently (same tolerance, deterministic).  Returns
    None (caller runs the full problem) when too few rows are ignored."""
    bt, h = x.shape
    dev = x.device
    limit = None
    if KEPT_ROWS_DEVICE_COUNT or torch.cuda.is_current_stream_capturing():
        # no host read: all bt row slots, kept rows first, ignored slots after (X rows 0,
        # targets ignore_index); the GEMMs skip the work past the device count
        kr = _take_prepared(t, ignore_index) if not torch.cuda.is_current_stream_capturing() else None
        if kr is not None:
            # the prepared compaction ran on another stream: order it before this one's readers
            kr.event.wait(torch.cuda.current_stream(dev))
            index, pos, limit = kr.index, kr.pos, kr.count
        else:
            index, pos, limit = _compact(t, ignore_index)
        n = bt
    else:
        kr = kept_rows(t, ignore_index)
        if kr is None:
            return None
        index, pos, n = kr
    # the kept targets are gathered here (8 bytes a row); the kept X rows are gathered by the
    # library one chunk at a time into its workspace (lk_flce_args.x_row_index), so no
    # n x H copy of X is ever held
    tk = _gather_rows(t, index, n, torch.empty(n, dtype=torch.int64, device=dev), int(ignore_index) & ((1 << 64) - 1))
    loss, z_loss, acc, pred, gxk, gw, gb = fused_linear_cross_entropy_forward(
        x, w, tk, compute_grad_input=need_gx, compute_grad_weight=need_gw, skip_ignored_rows=False,
        _x_row_index=index, _row_limit=limit, **kw)
    del tk
    gx = _gather_rows(gxk, pos, bt, torch.empty_like(x)) if gxk is not None else None
    if reduction == "none":  # per-row outputs back to every row (ignored: 0)
        loss = _gather_rows(loss, pos, bt, torch.empty(bt, dtype=loss.dtype, device=dev))
        if z_loss is not None:
            z_loss = _gather_rows(z_loss, pos, bt, torch.empty(bt, dtype=z_loss.dtype, device=dev))
        if acc is not None:
            acc = _gather_rows(acc, pos, bt, torch.empty(bt, dtype=acc.dtype, device=dev))
    if pred is not None:  # ignored rows predict -1 (LK/ops/cross_entropy.py:294-299)
        pred = _gather_rows(pred, pos, bt, torch.empty(bt, dtype=torch.int64, device=dev), (1 << 64) - 1)
    return loss, z_loss, acc, pred, gx, gw, gb


@device_guard
def fused_linear_cross_entropy_forward(
    _input: torch.Tensor,
    weight: torch.Tensor,
    target: torch.Tensor,
    ce_weight=None,
    bias: Optional[torch.Tensor] = None,
    ignore_index: int = -100,
    lse_square_scale: float = 0.0,
    label_smoothing: float = 0.0,
    reduction: str = "mean",
    softcap: Optional[float] = None,
    return_z_loss: bool = False,
    accum_dtype=None,
    use_token_scaling: bool = False,
    return_token_accuracy: bool = False,
    return_predicted_tokens: bool = False,
    chunk_rows: Optional[int] = None,
    force_simt: bool = False,
    compute_grad_input: Optional[bool] = None,
    compute_grad_weight: Optional[bool] = None,
    mean_count: Optional[torch.Tensor] = None,
    grad_w_slice_events=None,
    mean_weight_sum: Optional[torch.Tensor] = None,
    check_targets: bool = True,
    fp32_pieces: int = 0,
    grad_w_out: Optional[torch.Tensor] = None,
    skip_ignored_rows: Optional[bool] = None,
    _x_row_index: Optional[torch.Tensor] = None,
    _row_limit: Optional[torch.Tensor] = None,
):
    """Returns (loss, z_loss, token_accuracy, predicted_tokens, grad_input, grad_weight, grad_bias).

    Same return tuple as LK/ops/fused_linear_cross_entropy.py:17-244.  grad_weight across
    chunks (LK/ops/fused_linear_cross_entropy.py:64-69): accum_dtype=torch.float32 -> fp32
    workspace accumulator; accum_dtype=weight.dtype -> accumulated in the weight dtype
    (Liger's accum_dtype=None order, a TMA reduce-add in L2); accum_dtype=None -> the
    weight dtype when the plan has <= 8 chunks (no fp32 workspace: peak memory ~ one
    logits chunk), fp32 beyond that.  Returned in weight.dtype, as Liger does.
    `mean_count` (CUDA int64 scalar) overrides the MEAN denominator with a global
    non-ignored count (token-sharded mode).  `grad_w_slice_events` (list of torch.cuda.Event)
    splits the last chunk's grad_w GEMM into that many vocab-row slices and records event s
    when slice s of grad_w is final (overlap of the token-sharded dW all-reduce).
    fp32 inputs run on the bf16 tensor cores on split operands (`fp32_pieces` bf16 pieces
    per value: 0/3 = 6 piece products (fp32-exact products), 2 = 3; include/liger_b200.h);
    `force_simt=True` runs the SIMT FFMA GEMMs instead (the test reference).
    `check_targets=False` skips the host read of the device-side out-of-range count (the one
    host sync of the call); the caller then owns the check (token_sharded_flce does it on the
    all-reduced count after enqueueing its collectives).
    `grad_w_out` (contiguous, weight's shape / dtype / device) receives grad_weight instead of a
    new tensor: the token-sharded peer all-reduce passes a view of its symmetric buffer.
    `skip_ignored_rows` (default SKIP_IGNORED_ROWS) runs the chunk loop on the rows whose
    target is not ignore_index only (`_forward_kept_rows`); the outputs are those of the full
    call (ignored rows: loss 0, gradient 0, predicted token -1).  It costs one host read of the
    kept-row count, so the token-sharded (sync-free) path turns it off.
    """
    if not (0.0 <= label_smoothing <= 1.0):
        raise ValueError(f"label_smoothing must be between 0.0 and 1.0. Got: {label_smoothing}")
    if reduction not in _capi.REDUCTIONS:
        raise ValueError(f"reduction must be 'mean' or 'sum' or 'none'. Got: {reduction}")
    if softcap is not None and not softcap > 0:
        raise ValueError(f"softcap must greater than 0.0 or None. Got: {softcap}")
    require_cuda(_input, weight, target, bias)
    if _input.dim() != 2 or weight.dim() != 2:
        raise errors.ShapeMismatch("expected _input (BT, H) and weight (V, H)")
    bt, h = _input.shape
    if _x_row_index is not None:  # internal (_forward_kept_rows): the call's rows are x[_x_row_index[:n]]
        bt = target.numel()
    v, hw = weight.shape
    if hw != h:
        raise errors.ShapeMismatch(f"hidden width {h} != weight input width {hw}")
    if weight.dtype != _input.dtype:
        raise errors.ShapeMismatch(f"weight dtype {weight.dtype} != input dtype {_input.dtype}")
    if bias is not None and (bias.shape != (v,) or bias.dtype != weight.dtype):
        raise errors.ShapeMismatch("bias must be (V,) in the weight dtype")
    t = as_targets(target)
    if t.numel() != bt:
        raise errors.ShapeMismatch(f"need one target per row ({bt}), got {t.numel()}")
    x = _input.contiguous()
    w = weight.contiguous()
    b = bias.contiguous() if bias is not None else None
    require_contiguous("_input", x)
    need_gx = _input.requires_grad if compute_grad_input is None else compute_grad_input
    need_gw = (need_gx and weight.requires_grad) if compute_grad_weight is None else compute_grad_weight
    dev = x.device
    if (SKIP_IGNORED_ROWS if skip_ignored_rows is None else skip_ignored_rows) and bt >= COMPACT_MIN_SKIPPED:
        kept = _forward_kept_rows(
            x, w, t, ignore_index, need_gx, need_gw, reduction, return_z_loss, return_token_accuracy,
            return_predicted_tokens,
            dict(ce_weight=ce_weight, bias=b, ignore_index=ignore_index, lse_square_scale=lse_square_scale,
                 label_smoothing=label_smoothing, reduction=reduction, softcap=softcap, return_z_loss=return_z_loss,
                 accum_dtype=accum_dtype, use_token_scaling=use_token_scaling,
                 return_token_accuracy=return_token_accuracy, return_predicted_tokens=return_predicted_tokens,
                 chunk_rows=chunk_rows, force_simt=force_simt, mean_count=mean_count,
                 grad_w_slice_events=grad_w_slice_events, mean_weight_sum=mean_weight_sum,
                 check_targets=check_targets, fp32_pieces=fp32_pieces, grad_w_out=grad_w_out))
        if kept is not None:
            return kept
    grad_x = torch.empty(bt, h, dtype=x.dtype, device=dev) if need_gx else None
    if need_gw and grad_w_out is not None:
        if grad_w_out.shape != w.shape or grad_w_out.dtype != w.dtype or grad_w_out.device != w.device:
            raise errors.ShapeMismatch("grad_w_out must match weight's shape, dtype and device")
        require_contiguous("grad_w_out", grad_w_out)
    grad_w = (grad_w_out if grad_w_out is not None else torch.empty_like(w)) if need_gw else None
    grad_b = torch.empty_like(b) if (b is not None and need_gx) else None
    loss_rows = torch.empty(bt, dtype=torch.float32, device=dev)
    loss_sum = torch.empty((), dtype=torch.float32, device=dev)
    z_rows = torch.empty(bt, dtype=torch.float32, device=dev) if return_z_loss else None
    z_sum = torch.empty((), dtype=torch.float32, device=dev) if return_z_loss else None
    stats = torch.empty(2, dtype=torch.int64, device=dev)
    correct = torch.empty(bt, dtype=torch.float32, device=dev) if return_token_accuracy else None
    pred = torch.empty(bt, dtype=torch.int64, device=dev) if return_predicted_tokens else None
    cw = None
    if ce_weight is not None:  # Liger class weights (LK/ops/fused_linear_cross_entropy.py:86-98)
        if ce_weight.shape != (v,) or not torch.is_floating_point(ce_weight):
            raise errors.ShapeMismatch(f"ce_weight must be a floating tensor of size V={v}")
        cw = ce_weight.detach().to(device=dev, dtype=torch.float32).contiguous()
    L = lib()
    dt = dtype_code(x)
    cr = int(chunk_rows or 0)
    if fp32_pieces not in (0, 2, 3):
        raise ValueError(f"fp32_pieces must be 0 (default), 2 or 3. Got: {fp32_pieces}")
    if force_simt:
        accum = _capi.LK_ACCUM_FP32  # the SIMT (fp32 parity) GEMM accumulates dW in an fp32 workspace
    elif accum_dtype is None:
        accum = _capi.LK_ACCUM_AUTO
    elif accum_dtype == torch.float32:
        accum = _capi.LK_ACCUM_FP32
    elif accum_dtype == weight.dtype:
        accum = _capi.LK_ACCUM_WEIGHT_DTYPE
    else:
        raise errors.UnsupportedOption(f"accum_dtype {accum_dtype}: use None, torch.float32 or the weight dtype")
    args = _capi.FlceArgs(
        x=ptr(x), weight=ptr(w), target=ptr(t), bias=ptr(b), bt=bt, hidden=h, vocab=v, dtype=dt,
        x_row_index=ptr(_x_row_index), row_limit=ptr(_row_limit),
        ignore_index=int(ignore_index), label_smoothing=float(label_smoothing),
        lse_square_scale=float(lse_square_scale), softcap=float(softcap) if softcap is not None else 0.0,
        reduction=_capi.REDUCTIONS[reduction], chunk_rows=cr, loss_rows=ptr(loss_rows), loss_sum=ptr(loss_sum),
        z_loss_rows=ptr(z_rows), z_loss_sum=ptr(z_sum), grad_x=ptr(grad_x), grad_w=ptr(grad_w),
        grad_bias=ptr(grad_b), target_stats=ptr(stats), workspace=None, workspace_bytes=0,
        stream=stream_of(x), force_simt=int(bool(force_simt)), fp32_pieces=int(fp32_pieces or 0),
        mean_count=ptr(mean_count) if mean_count is not None else None, grad_w_accum=accum,
        token_correct_rows=ptr(correct), predicted_tokens=ptr(pred), use_token_scaling=int(bool(use_token_scaling)),
        ce_weight=ptr(cw),
        mean_weight_sum=ptr(mean_weight_sum) if mean_weight_sum is not None else None,
    )
    ws = workspace(L.lk_flce_workspace_bytes_for(_capi.C.byref(args)), dev)  # sized for exactly this call
    args.workspace, args.workspace_bytes = ptr(ws), ws.numel()
    ev_arr = None
    if grad_w_slice_events:
        for ev in grad_w_slice_events:  # torch creates the CUDA event lazily on first record
            if not ev.cuda_event:
                ev.record(torch.cuda.current_stream(dev))
        ev_arr = (_capi.C.c_void_p * len(grad_w_slice_events))(*[ev.cuda_event for ev in grad_w_slice_events])
        args.grad_w_slices = len(grad_w_slice_events)
        args.grad_w_slice_events = _capi.C.cast(ev_arr, _capi.C.c_void_p)
    if mean_count is not None and (mean_count.dtype != torch.int64 or not mean_count.is_cuda):
        raise errors.ShapeMismatch("mean_count must be a CUDA int64 tensor")
    if mean_weight_sum is not None and (mean_weight_sum.dtype != torch.float32 or not mean_weight_sum.is_cuda):
        raise errors.ShapeMismatch("mean_weight_sum must be a CUDA float32 tensor")
    # the range check reads a count staged ahead of the GEMMs: the host waits for that count
    # kernel only, and runs ahead to the next op while this one computes
    staged = count_and_stage_targets(t, v, int(ignore_index)) if check_targets else None
    check(L.lk_flce_forward_backward(_capi.C.byref(args)))
    del ws
    raise_if_staged_out_of_range(staged, v)
    if reduction == "none":
        loss = loss_rows
        z_loss = z_rows.to(x.dtype) if return_z_loss else None
        acc = correct
    else:
        loss = loss_sum
        z_loss = z_sum.to(x.dtype) if return_z_loss else None
        acc = None
        if return_token_accuracy:  # mean over non-ignored tokens (LK/ops/fused_linear_cross_entropy.py:234-236)
            denom = (mean_count[:1] if mean_count is not None else stats[:1]).clamp(min=1)
            acc = correct.sum() / denom[0]
    return loss, z_loss, acc, pred, grad_x, grad_w, grad_b


@device_guard
def fused_linear_cross_entropy_backward(grad_output, grad_input, grad_weight, grad_bias):
    """Scale the forward-computed gradients by grad_output (LK/ops/fused_linear_cross_entropy.py:247-291).

    The scale kernel reads grad_output on the device and returns immediately when it
    is 1.0, so there is no torch.equal host sync.
    """
    if grad_output.ndim > 0:
        g = grad_output.reshape(-1)
        # dW = sum_r g_r dZ_r^T x_r cannot be rescaled after the fact unless g is uniform.
        if g.numel() and not bool(torch.all(g == g[0])):
            raise errors.UnsupportedOption("reduction='none' backward with a non-uniform grad_output")
        g = g[:1] if g.numel() else torch.ones(1, device=grad_output.device)
    else:
        g = grad_output.reshape(1)
    g = g.detach().to(torch.float32).contiguous()
    L = lib()
    for t in (grad_input, grad_weight):
        if t is not None and t.numel():
            check(L.lk_scale_by_device_scalar(t.data_ptr(), t.shape[0], t.shape[1], t.stride(0), dtype_code(t),
                                              g.data_ptr(), stream_of(t)))
    if grad_bias is not None and grad_bias.numel():
        check(L.lk_scale_by_device_scalar(grad_bias.data_ptr(), 1, grad_bias.numel(), grad_bias.numel(),
                                          dtype_code(grad_bias), g.data_ptr(), stream_of(grad_bias)))
    return grad_input, grad_weight, grad_bias


class LigerFusedLinearCrossEntropyFunction(torch.autograd.Function):
    """Same signature and 15-slot backward arity as LK/ops/fused_linear_cross_entropy.py:294-400."""

    @staticmethod
    def forward(
        ctx,
        _input,
        weight,
        target,
        bias=None,
        ce_weight=None,
        ignore_index=-100,
        lse_square_scale=0.0,
        label_smoothing=0.0,
        reduction="mean",
        softcap=None,
        return_z_loss: bool = False,
        accum_dtype=None,
        use_token_scaling: bool = False,
        return_token_accuracy: bool = False,
        return_predicted_tokens: bool = False,
        chunk_rows: Optional[int] = None,
    ):
        loss, z_loss, acc, pred, gx, gw, gb = fused_linear_cross_entropy_forward(
            _input, weight, target, ce_weight, bias, ignore_index, lse_square_scale, label_smoothing, reduction,
            softcap, return_z_loss, accum_dtype, use_token_scaling, return_token_accuracy,
            return_predicted_tokens, chunk_rows=chunk_rows,
        )
        ctx.save_for_backward(
            gx.detach() if gx is not None else None,
            gw.detach() if gw is not None else None,
            gb.detach() if gb is not None else None,
        )
        return loss, z_loss, acc, pred

    @staticmethod
    def backward(ctx, grad_output, grad_output2, grad_output3, grad_output4):
        gx, gw, gb = ctx.saved_tensors
        gx, gw, gb = fused_linear_cross_entropy_backward(grad_output, gx, gw, gb)
        return (gx, gw, None, gb) + (None,) * 12


class LigerFusedLinearCrossEntropyLoss(torch.nn.Module):
    """Drop-in for LK/transformers/fused_linear_cross_entropy.py:9-69 (plus an optional chunk_rows override)."""

    def __init__(
        self,
        ce_weight: Optional[torch.FloatTensor] = None,
        ignore_index: int = -100,
        lse_square_scale: float = 0.0,
        label_smoothing: float = 0.0,
        reduction: str = "mean",
        softcap: Optional[float] = None,
        return_z_loss: bool = False,
        accum_dtype: Optional[torch.dtype] = None,
        use_token_scaling: bool = False,
        return_token_accuracy: bool = False,
        return_predicted_tokens: bool = False,
        chunk_rows: Optional[int] = None,
    ):
        super().__init__()
        assert 0 <= label_smoothing <= 1, f"label_smoothing must be between 0.0 and 1.0. Got: {label_smoothing}"
        assert reduction in {"mean", "sum", "none"}, f"reduction must be 'mean' or 'sum' or 'none'. Got: {reduction}"
        assert softcap is None or softcap > 0, f"softcap must greater than 0.0 or None. Got: {softcap}"
        self.ce_weight = ce_weight
        self.ignore_index = ignore_index
        self.lse_square_scale = lse_square_scale
        self.label_smoothing = label_smoothing
        self.reduction = reduction
        self.softcap = softcap
        self.return_z_loss = return_z_loss
        self.accum_dtype = accum_dtype
        self.use_token_scaling = use_token_scaling
        self.return_token_accuracy = return_token_accuracy
        self.return_predicted_tokens = return_predicted_tokens
        self.chunk_rows = chunk_rows

    def forward(self, lin_weight, _input, target, bias=None):
        loss, z_loss, acc, pred = LigerFusedLinearCrossEntropyFunction.apply(
            _input, lin_weight, target, bias, self.ce_weight, self.ignore_index, self.lse_square_scale,
            self.label_smoothing, self.reduction, self.softcap, self.return_z_loss, self.accum_dtype,
            self.use_token_scaling, self.return_token_accuracy, self.return_predicted_tokens, self.chunk_rows,
        )
        if not self.return_z_loss and not self.return_token_accuracy and not self.return_predicted_tokens:
            return loss
        return CrossEntropyOutput(loss=loss, z_loss=z_loss, token_accuracy=acc, predicted_tokens=pred)
