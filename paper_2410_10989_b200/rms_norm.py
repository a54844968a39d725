"""RMSNorm: LigerRMSNormFunction / LigerRMSNorm.

Drop-in for LK/transformers/rms_norm.py:7-46 and LK/ops/rms_norm.py:581-666;
math of rowfuse/ops.py:190-241 (one cached rstd per row, x-hat recomputed in the
backward, deterministic two-stage dW).  Casting modes 'llama' / 'gemma' / 'none'
and the weight offset follow Liger.
"""

from __future__ import annotations

import torch
import torch.nn as nn

from . import _capi
from ._utils import check, device_guard, dtype_code, lib, ptr, require_cuda, stream_of, workspace


@device_guard
def rms_norm_forward(X, W, eps, offset=0.0, casting_mode="llama"):
    require_cuda(X, W)
    mode = _capi.CASTING[casting_mode] if isinstance(casting_mode, str) else int(casting_mode)
    shape = X.shape
    X2 = X.reshape(-1, shape[-1]).contiguous()
    rows, cols = X2.shape
    if W is not None and (W.shape != (cols,)):
        raise ValueError("Incompatible hidden size dimension between input tensor and weight")
    # The kernels read the weight in the activation dtype: a weight of another dtype (e.g. fp32
    # weight with bf16 activations, which Liger accepts) is cast first, as layer_norm.py does.
    Wc = W.to(X2.dtype).contiguous() if W is not None else None
    Y = torch.empty_like(X2)
    rstd = torch.empty(rows, dtype=torch.float32 if mode in (0, 1) else X2.dtype, device=X2.device)
    check(lib().lk_rmsnorm_fwd(ptr(X2), ptr(Wc), ptr(Y), ptr(rstd), rows, cols, float(eps), float(offset), mode,
                               dtype_code(X2), stream_of(X2)))
    return Y.view(shape), X2, rstd, mode


@device_guard
def rms_norm_backward(dY, X2, W, rstd, offset, mode, in_place):
    shape = dY.shape
    dY2 = dY.reshape(-1, shape[-1]).contiguous()
    rows, cols = dY2.shape
    dX = dY2 if in_place else torch.empty_like(dY2)
    w_dtype = W.dtype if W is not None else None
    if W is not None and W.dtype != dY2.dtype:
        W = W.to(dY2.dtype)
    dW = torch.empty_like(W) if W is not None else None
    L = lib()
    ws = workspace(L.lk_rmsnorm_bwd_workspace_bytes(rows, cols), dY2.device) if W is not None else None
    check(L.lk_rmsnorm_bwd(ptr(dY2), ptr(X2), ptr(W), ptr(rstd), ptr(dX), ptr(dW), rows, cols, float(offset), mode,
                           dtype_code(dY2), ptr(ws), ws.numel() if ws is not None else 0, stream_of(dY2)))
    if dW is not None and dW.dtype != w_dtype:
        dW = dW.to(w_dtype)  # Liger returns dW in the weight's dtype
    return dX.view(shape), dW


class LigerRMSNormFunction(torch.autograd.Function):
    """forward(X, W, eps, offset=0.0, casting_mode='llama', in_place=True, row_mode=None)."""

    @staticmethod
    def forward(ctx, X, W, eps, offset=0.0, casting_mode="llama", in_place=True, row_mode=None):
        Y, X2, rstd, mode = rms_norm_forward(X, W, eps, offset, casting_mode)
        ctx.offset = offset
        ctx.mode = mode
        ctx.in_place = in_place
        ctx.has_w = W is not None
        if W is not None:
            ctx.save_for_backward(X2, W.contiguous(), rstd)
        else:
            ctx.save_for_backward(X2, rstd)
        return Y

    @staticmethod
    def backward(ctx, dY):
        if ctx.has_w:
            X2, W, rstd = ctx.saved_tensors
        else:
            (X2, rstd), W = ctx.saved_tensors, None
        dX, dW = rms_norm_backward(dY, X2, W, rstd, ctx.offset, ctx.mode, ctx.in_place)
        return dX, dW, None, None, None, None, None


class LigerRMSNorm(nn.Module):
    """Drop-in for LK/transformers/rms_norm.py:7-46."""

    def __init__(self, hidden_size, eps=1e-6, offset=0.0, casting_mode="llama", init_fn="ones", in_place=True,
                 row_mode=None, elementwise_affine=True):
        super().__init__()
        assert init_fn in ["ones", "zeros"], f"init_fn must be either 'ones' or 'zeros', got {init_fn}"
        self.elementwise_affine = elementwise_affine
        if elementwise_affine:
            self.weight = nn.Parameter(torch.ones(hidden_size) if init_fn == "ones" else torch.zeros(hidden_size))
        else:
            self.register_parameter("weight", None)
        self.variance_epsilon, self.offset, self.casting_mode, self.in_place, self.row_mode = (
            eps, offset, casting_mode, in_place, row_mode)

    def forward(self, hidden_states):
        return LigerRMSNormFunction.apply(hidden_states, self.weight, self.variance_epsilon, self.offset,
                                          self.casting_mode, self.in_place, self.row_mode)

    def extra_repr(self):
        return f"weight_shape={tuple(self.weight.shape) if self.weight is not None else None}, eps={self.variance_epsilon}, offset={self.offset}, in_place={self.in_place}"
