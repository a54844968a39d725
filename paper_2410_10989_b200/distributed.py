"""Multi-GPU FLCE: token-sharded and vocab-parallel modes (one process per GPU).

Token-sharded.  Rank r owns rows [r*BT/R, (r+1)*BT/R) and a
full replica of W.  Rows are independent except for the MEAN denominator and the
dW sum (rowfuse/flce.py:161-168; dW additivity over row groups is the reference's
own test, tests/test_flce.py:182-205).  Collectives: one int64 all-reduce of the
non-ignored count before the local FLCE (so every rank divides by the global
count inside the finalize kernel, no host sync), one all-reduce of the loss, one
NCCL all-reduce of dW in the weight dtype.

Vocab-parallel (row 2).  Rank r owns W rows [v0, v0 + V/R) and sees all tokens.
Per row chunk: local logits + per-row (max, sumexp, sum_logits, target_logit)
statistics (lk_flce_vp_logits), an all-reduce of the statistics (MAX, then SUM
of rescaled sums), then local dlogits, an fp32 partial dX (all-reduced SUM) and
the local dW shard (no communication) (lk_flce_vp_backward).

The compute callbacks are injectable so the host-side collective logic is tested
on CPU with gloo and the oracle standing in for the CUDA kernels
(tests/test_distributed.py); the default callbacks are the sm_100a library.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist

from . import _capi
from ._utils import (
    as_targets,
    check,
    device_guard,
    dtype_code,
    lib,
    ptr,
    raise_if_staged_out_of_range,
    stage_target_stats,
    stream_of,
    workspace,
)


# ------------------------------------------------------------- token sharded
def shard_rows(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, as-even-as-possible row range of `rank`."""
    base, extra = divmod(n_rows, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@device_guard
def _count_cuda(t: torch.Tensor, vocab: int, ignore_index: int) -> torch.Tensor:
    out = torch.empty(2, dtype=torch.int64, device=t.device)
    check(lib().lk_count_targets(t.data_ptr(), t.numel(), vocab, ignore_index, out.data_ptr(), stream_of(t)))
    return out


MAX_DW_SLICES = 16  # LK_MAX_GRAD_W_SLICES (include/liger_b200.h)


def _local_flce_cuda(x, w, t, mean_count, reduction="mean", **kw):
    from .fused_linear_cross_entropy import fused_linear_cross_entropy_forward

    # no host read of the out-of-range count here: token_sharded_flce checks the GLOBAL count
    # after every collective is enqueued, so the dW all-reduce can overlap the dW GEMMs
    loss, _, _, _, gx, gw, _ = fused_linear_cross_entropy_forward(
        x, w, t, compute_grad_input=True, compute_grad_weight=True, reduction=reduction,
        mean_count=mean_count[:1] if reduction == "mean" else None, check_targets=False, **kw)
    return loss, gx, gw


_COMM_STREAMS: dict = {}


def _comm_stream(device: torch.device) -> torch.cuda.Stream:
    """One side stream per device for the overlapped grad_w all-reduce (created once)."""
    key = torch.device(device).index
    if key not in _COMM_STREAMS:
        _COMM_STREAMS[key] = torch.cuda.Stream(device=device)
    return _COMM_STREAMS[key]


def _allreduce_grad_w_overlapped(x, w, t, counts, group, dw_slices, local_fn, kw, peer=None):
    """Local FLCE whose last-chunk grad_w GEMM is split into `dw_slices` vocab-row slices;
    slice s is all-reduced on a side stream as soon as its event fires, so all but the last
    slice's all-reduce hide under the remaining dW GEMM launches.  The library records every
    event on every path (include/liger_b200.h, grad_w_slice_events), so a slice is never
    all-reduced before it is final -- also on the SIMT path or for a rank with no rows.
    With `peer` (a PeerBuffer) grad_w lives in the symmetric buffer and each slice is summed by
    the peer-memory kernel (lk_peer_allreduce) instead of NCCL."""
    events = [torch.cuda.Event() for _ in range(dw_slices)]
    if peer is not None:
        kw = dict(kw, grad_w_out=peer.tensor(w.shape, w.dtype))
    loss, gx, gw = local_fn(x, w, t, counts, grad_w_slice_events=events, **kw)
    v, h = gw.shape
    step = -(-v // dw_slices)
    rows = -(-step // 256) * 256  # same slice bounds as the library (flce.cu)
    comm = _comm_stream(gw.device)
    for s, ev in enumerate(events):
        lo, hi = s * rows, min(v, (s + 1) * rows)
        comm.wait_event(ev)
        if lo < hi:
            if peer is not None:
                peer.all_reduce_(gw, lo * h, hi * h, stream=comm)
            else:
                with torch.cuda.stream(comm):
                    dist.all_reduce(gw[lo:hi], op=dist.ReduceOp.SUM, group=group)
    torch.cuda.current_stream(gw.device).wait_stream(comm)
    if peer is None:
        gw.record_stream(comm)
    return loss, gx, gw


def token_sharded_flce(
    x_local: torch.Tensor,
    weight: torch.Tensor,
    target_local: torch.Tensor,
    group=None,
    ignore_index: int = -100,
    reduction: str = "mean",
    count_fn: Optional[Callable] = None,
    local_fn: Optional[Callable] = None,
    reduce_grad_weight: bool = True,
    dw_slices: int = 4,
    check_targets: bool = True,
    comm: str = "nccl",
    skip_ignored_rows: Optional[bool] = None,
    **kw,
):
    """Returns (loss, local grad_x, all-reduced grad_w).

    `loss` is the global scalar for reduction 'mean'/'sum'; for 'none' it is this rank's
    per-row loss vector (rows of different ranks are not summed element-wise).
    With the CUDA kernels (default `local_fn`) and 2 <= `dw_slices` <= 16, the grad_w
    all-reduce overlaps the last chunk's grad_w GEMM (`_allreduce_grad_w_overlapped`): the
    call enqueues every kernel and collective without a host sync (see skip_ignored_rows below),
    and only then (with
    `check_targets`) reads the globally all-reduced out-of-range target count, so every rank
    raises TargetOutOfRange together instead of one rank leaving the others in a collective.
    The local FLCE skips this rank's ignore_index rows (`skip_ignored_rows`, default
    SKIP_IGNORED_ROWS: fused_linear_cross_entropy._forward_kept_rows).  That costs one host read
    of the kept-row count at the start of the local call, before its GEMMs, so the dW overlap
    is unaffected; `skip_ignored_rows=False` keeps the call entirely free of host reads.
    `comm="peer"` sums grad_w with the peer-memory kernel over a symmetric buffer
    (peer.grad_w_buffer, csrc/peer.cu) instead of NCCL; the returned grad_w is then a view of
    that buffer, overwritten by the next call for the same weight shape.
    """
    if reduction not in ("mean", "sum", "none"):
        raise ValueError(f"reduction must be 'mean' or 'sum' or 'none'. Got: {reduction}")
    if comm not in ("nccl", "peer"):
        raise ValueError(f"comm must be 'nccl' or 'peer'. Got: {comm}")
    t = as_targets(target_local) if target_local.is_cuda else target_local.reshape(-1).to(torch.int64)
    count_fn = count_fn or (lambda tt: _count_cuda(tt, weight.shape[0], ignore_index))
    dw_slices = max(1, min(int(dw_slices), MAX_DW_SLICES))
    overlap = local_fn is None and reduce_grad_weight and dw_slices > 1 and x_local.is_cuda
    cuda_local = local_fn is None
    local_fn = local_fn or _local_flce_cuda
    counts = count_fn(t)
    # (n_valid, n_out_of_range) summed over ranks: the MEAN denominator and the global range check
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    staged = stage_target_stats(counts) if (check_targets and cuda_local) else None
    kw = dict(kw, ignore_index=ignore_index, reduction=reduction)
    if cuda_local:
        kw["skip_ignored_rows"] = skip_ignored_rows
    cw = kw.get("ce_weight")
    if cw is not None and reduction == "mean" and local_fn is _local_flce_cuda:
        # weighted MEAN: the denominator is the GLOBAL sum of the valid targets' weights
        valid = (t != ignore_index) & (t >= 0) & (t < cw.numel())
        wsum = cw.detach().to(device=t.device, dtype=torch.float32)[t.clamp(0, cw.numel() - 1)]
        wsum = (wsum * valid).sum(dtype=torch.float32).reshape(1)
        dist.all_reduce(wsum, op=dist.ReduceOp.SUM, group=group)
        kw["mean_weight_sum"] = wsum
    peer = None
    if comm == "peer" and reduce_grad_weight and cuda_local and x_local.is_cuda:
        from .peer import grad_w_buffer

        peer = grad_w_buffer(weight, group)
    if overlap or peer is not None:
        loss, gx, gw = _allreduce_grad_w_overlapped(x_local, weight, t, counts, group, dw_slices, local_fn, kw,
                                                    peer=peer)
    else:
        loss, gx, gw = local_fn(x_local, weight, t, counts, **kw)
        if reduce_grad_weight and gw is not None:
            dist.all_reduce(gw, op=dist.ReduceOp.SUM, group=group)
    if reduction != "none":
        loss = loss.clone()
        dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)
    if check_targets and cuda_local:
        raise_if_staged_out_of_range(staged, weight.shape[0])
        if peer is not None:
            peer.check()
    return loss, gx, gw


# ------------------------------------------------------------ vocab parallel
@dataclass
class VocabShard:
    offset: int
    size: int
    total: int


def vocab_shard(vocab: int, rank: int, world: int) -> VocabShard:
    lo, hi = shard_rows(vocab, rank, world)
    return VocabShard(lo, hi - lo, vocab)


def combine_row_stats(stats: torch.Tensor, ops, group=None) -> torch.Tensor:
    """Global per-row (max, sumexp, sum_logits, target_logit) across vocab shards: ONE
    all_gather of the [rows, 4] local statistics, then `ops.combine_stats` folds the ranks in
    rank order (lk_flce_vp_combine_stats), so every rank holds bit-identical statistics."""
    world = dist.get_world_size(group)
    rows = stats.shape[0]
    gathered = torch.empty(world * rows, stats.shape[1], dtype=stats.dtype, device=stats.device)
    dist.all_gather_into_tensor(gathered, stats.contiguous(), group=group)
    return ops.combine_stats(gathered.view(world, rows, stats.shape[1]))


class CudaVocabOps:
    """Default stage implementations: the sm_100a library."""

    def __init__(self, dtype: torch.dtype, device: torch.device):
        self.dt = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}[dtype]
        self.device = device

    def logits_stats(self, x, w_shard, t, shard: VocabShard, softcap, ignore_index):
        rows, h = x.shape
        ldz = -(-shard.size // 64) * 64
        buf = torch.empty(rows, ldz, dtype=x.dtype, device=x.device)
        stats = torch.empty(rows, 4, dtype=torch.float32, device=x.device)
        L = lib()
        ws = workspace(L.lk_flce_vp_workspace_bytes(rows, h, shard.size, self.dt), x.device)
        check(L.lk_flce_vp_logits(ptr(x), ptr(w_shard), ptr(t), rows, h, shard.size, shard.offset, self.dt,
                                  ignore_index, float(softcap or 0.0), ptr(stats), ptr(buf), ptr(ws), ws.numel(),
                                  stream_of(x)))
        return stats, buf

    def combine_stats(self, gathered):
        world, rows = gathered.shape[0], gathered.shape[1]
        out = torch.empty(rows, 4, dtype=torch.float32, device=gathered.device)
        check(lib().lk_flce_vp_combine_stats(ptr(gathered), world, rows, ptr(out), stream_of(gathered)))
        return out

    def backward(self, x, w_shard, t, shard, stats_g, buf, n_valid, gw_acc, accumulate, *, ignore_index,
                 label_smoothing, lse_square_scale, softcap, reduction, gx_out=None):
        """dX partial into `gx_out` (the x dtype or fp32) when given, else a new fp32 tensor."""
        rows, h = x.shape
        loss_rows = torch.empty(rows, dtype=torch.float32, device=x.device)
        gx = gx_out if gx_out is not None else torch.empty(rows, h, dtype=torch.float32, device=x.device)
        ws = workspace(256, x.device)
        check(lib().lk_flce_vp_backward2(
            ptr(x), ptr(w_shard), ptr(t), rows, h, shard.size, shard.offset, shard.total, self.dt, ignore_index,
            float(label_smoothing), float(lse_square_scale), float(softcap or 0.0), _capi.REDUCTIONS[reduction],
            ptr(n_valid), ptr(stats_g), ptr(buf), ptr(loss_rows), ptr(gx), dtype_code(gx), ptr(gw_acc),
            dtype_code(gw_acc), int(accumulate), ptr(ws), ws.numel(), stream_of(x)))
        return loss_rows, gx

    def count(self, t, vocab, ignore_index):
        return _count_cuda(t, vocab, ignore_index)


@device_guard
def vocab_parallel_flce(
    x: torch.Tensor,
    w_shard: torch.Tensor,
    target: torch.Tensor,
    shard: VocabShard,
    group=None,
    ignore_index: int = -100,
    label_smoothing: float = 0.0,
    lse_square_scale: float = 0.0,
    softcap: Optional[float] = None,
    reduction: str = "mean",
    chunk_rows: int = 2048,
    ops=None,
    accum_dtype: Optional[torch.dtype] = None,
    dx_reduce_dtype: Optional[torch.dtype] = None,
    check_targets: bool = True,
    skip_ignored_rows: Optional[bool] = None,
    comm: str = "nccl",
    _x_row_index: Optional[torch.Tensor] = None,
):
    """Returns (loss, grad_x (all-reduced, x dtype), local grad_w shard (w dtype)).

    Every rank holds all rows of x and the targets; only W is sharded by vocab rows.
    `accum_dtype` follows Liger's FLCE option: None accumulates the dW shard across chunks
    in the weight dtype (16-bit weights), torch.float32 in an fp32 buffer.
    The dX partial of chunk k is all-reduced asynchronously (`async_op=True`) while chunk k+1
    computes; by default it is written by the backward GEMM straight into grad_x in the x
    dtype and reduced there in place (`dx_reduce_dtype=torch.float32` reduces fp32 partials
    and casts after the last wait).  The only wait is on the outstanding reductions at the end.
    With the CUDA ops the ignore_index rows are skipped (`skip_ignored_rows`, default
    SKIP_IGNORED_ROWS): every rank holds the same targets, so every rank compacts the same rows
    and the collectives stay matched; one host read of the kept-row count.
    `comm="peer"` sums each chunk's dX partial with the peer-memory kernel (csrc/peer.cu) over
    a symmetric grad_x buffer instead of NCCL (x-dtype reduction only); the returned grad_x is
    then a view of that buffer, overwritten by the next call of the same shape.
    """
    if comm not in ("nccl", "peer"):
        raise ValueError(f"comm must be 'nccl' or 'peer'. Got: {comm}")
    from . import fused_linear_cross_entropy as flce_mod

    skip = flce_mod.SKIP_IGNORED_ROWS if skip_ignored_rows is None else skip_ignored_rows
    if ops is None and skip and x.is_cuda:
        t_all = target.reshape(-1).to(torch.int64).contiguous()
        kr = flce_mod.kept_rows(t_all, ignore_index)
        if kr is not None:
            index, pos, n = kr
            bt_all, h = x.shape
            tk = flce_mod._gather_rows(t_all, index, n, torch.empty(n, dtype=torch.int64, device=x.device))
            # X rows are gathered chunk by chunk inside the loop (_x_row_index): no n x H copy
            loss, gxk, gw = vocab_parallel_flce(
                x.contiguous(), w_shard, tk, shard, group=group, ignore_index=ignore_index,
                label_smoothing=label_smoothing, lse_square_scale=lse_square_scale, softcap=softcap,
                reduction=reduction, chunk_rows=chunk_rows, accum_dtype=accum_dtype, dx_reduce_dtype=dx_reduce_dtype,
                check_targets=check_targets, skip_ignored_rows=False, comm=comm, _x_row_index=index)
            gx = flce_mod._gather_rows(gxk, pos, bt_all, torch.empty(bt_all, h, dtype=x.dtype, device=x.device))
            if reduction == "none":
                loss = flce_mod._gather_rows(loss, pos, bt_all,
                                             torch.empty(bt_all, dtype=loss.dtype, device=x.device))
            return loss, gx, gw
    ops = ops or CudaVocabOps(x.dtype, x.device)
    t = target.reshape(-1).to(torch.int64).contiguous()
    bt, h = x.shape
    if _x_row_index is not None:  # internal (kept rows): the call's rows are x[_x_row_index[:len(t)]]
        bt = t.numel()
    n_valid = ops.count(t, shard.total, ignore_index)
    staged = stage_target_stats(n_valid) if (check_targets and isinstance(ops, CudaVocabOps)) else None
    if w_shard.dtype == torch.float64:
        acc_dtype = torch.float64
    elif accum_dtype is None and w_shard.dtype in (torch.bfloat16, torch.float16) and isinstance(ops, CudaVocabOps):
        acc_dtype = w_shard.dtype  # in-place weight-dtype accumulation (lk_flce_vp_backward_ex)
    else:
        acc_dtype = torch.float32
    gw_acc = torch.zeros(shard.size, h, dtype=acc_dtype, device=x.device)
    dx_dt = dx_reduce_dtype or x.dtype
    peer = None
    if comm == "peer" and isinstance(ops, CudaVocabOps) and dx_dt == x.dtype:
        from .peer import buffer_for

        # sized for all of x's rows (the kept-row call uses a prefix): one buffer per batch shape
        peer = buffer_for(x.shape[0] * h * x.element_size(), x.device, group, "vp_grad_x")
        gx = peer.tensor((bt, h), x.dtype)
        comm_stream = _comm_stream(x.device)
    else:
        gx = torch.empty(bt, h, dtype=x.dtype, device=x.device)
    loss_rows = torch.empty(bt, dtype=torch.float32, device=x.device)
    kw = dict(ignore_index=ignore_index, label_smoothing=label_smoothing, lse_square_scale=lse_square_scale,
              softcap=softcap, reduction=reduction)
    pending = []  # (work, lo, hi, partial) of in-flight dX reductions
    for ci, lo in enumerate(range(0, bt, chunk_rows)):
        hi = min(lo + chunk_rows, bt)
        if _x_row_index is not None:
            xc = flce_mod._gather_rows(x, _x_row_index[lo:hi], hi - lo,
                                       torch.empty(hi - lo, h, dtype=x.dtype, device=x.device))
        else:
            xc = x[lo:hi].contiguous()
        tc = t[lo:hi]
        stats, buf = ops.logits_stats(xc, w_shard, tc, shard, softcap, ignore_index)
        stats_g = combine_row_stats(stats, ops, group)
        gx_out = gx[lo:hi] if dx_dt == x.dtype else torch.empty(hi - lo, h, dtype=dx_dt, device=x.device)
        lr, gxp = ops.backward(xc, w_shard, tc, shard, stats_g, buf, n_valid, gw_acc, ci > 0, gx_out=gx_out, **kw)
        if peer is not None:  # this chunk's dX rows summed over peer memory on the side stream
            comm_stream.wait_stream(torch.cuda.current_stream(x.device))
            peer.all_reduce_(gx, lo * h, hi * h, stream=comm_stream)
        else:
            pending.append((dist.all_reduce(gxp, op=dist.ReduceOp.SUM, group=group, async_op=True), lo, hi, gxp))
        loss_rows[lo:hi] = lr
    if peer is not None:
        torch.cuda.current_stream(x.device).wait_stream(comm_stream)
    for work, lo, hi, gxp in pending:
        work.wait()
        if gxp.data_ptr() != gx[lo:hi].data_ptr():
            gx[lo:hi] = gxp.to(x.dtype)
    loss = loss_rows if reduction == "none" else loss_rows.sum()
    if check_targets and isinstance(ops, CudaVocabOps):
        raise_if_staged_out_of_range(staged, shard.total)
        if peer is not None:
            peer.check()
    return loss, gx, gw_acc.to(w_shard.dtype)
