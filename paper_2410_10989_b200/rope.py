"""RoPE: LigerRopeFunction / liger_rotary_pos_emb.

Drop-in for LK/transformers/rope.py:8-24 and LK/ops/rope.py:115-260: q and k
arrive as (bsz, n_head, seq, head_dim) views of (bsz, seq, n_head, head_dim)
storage, are rotated in place by the sm_100a kernel and returned as the same
transposed views.  Half-split rotation of rowfuse/ops.py:322-382.
"""

from __future__ import annotations

import torch

from . import errors
from ._utils import check, device_guard, dtype_code, lib, require_cuda, stream_of


@device_guard
def _rope(q, k, cos, sin, backward: bool):
    require_cuda(q, k, cos, sin)
    qt = q.transpose(1, 2).contiguous()  # physical (B, T, nq, d); no-op for HF layouts
    kt = k.transpose(1, 2).contiguous()
    b, t, nq, d = qt.shape
    nk = kt.shape[2]
    if kt.shape[0] != b or kt.shape[1] != t or kt.shape[3] != d:
        raise errors.ShapeMismatch("q and k must share batch, seq_len and head_dim")
    if cos.dim() == 2:
        cos, sin = cos.unsqueeze(0), sin.unsqueeze(0)
    cos = cos.contiguous()
    sin = sin.contiguous()
    if cos.shape[-2] != t or cos.shape[-1] != d or cos.shape != sin.shape:
        raise errors.ShapeMismatch(f"cos/sin must be (1 or B, {t}, {d}), got {tuple(cos.shape)}")
    check(lib().lk_rope(qt.data_ptr(), kt.data_ptr(), cos.data_ptr(), sin.data_ptr(), b, t, nq, nk, d,
                        cos.shape[0], dtype_code(qt), dtype_code(cos), int(backward), stream_of(qt)))
    return qt.transpose(1, 2), kt.transpose(1, 2), cos, sin


class LigerRopeFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, cos, sin, position_ids=None, unsqueeze_dim=1):
        q, k, cos, sin = _rope(q, k, cos, sin, backward=False)
        ctx.save_for_backward(cos, sin)
        return q, k

    @staticmethod
    def backward(ctx, dq, dk):
        cos, sin = ctx.saved_tensors
        dq, dk, _, _ = _rope(dq, dk, cos, sin, backward=True)
        return dq, dk, None, None, None, None


def liger_rotary_pos_emb(q, k, cos, sin, position_ids=None, unsqueeze_dim=1):
    """Apply RoPE to q (bsz, n_q_head, seq, d) and k (bsz, n_kv_head, seq, d)."""
    return LigerRopeFunction.apply(q, k, cos, sin, position_ids, unsqueeze_dim)
