"""LayerNorm: LigerLayerNormFunction / LigerLayerNorm.

Drop-in for LK/transformers/layer_norm.py:7-25 and LK/ops/layer_norm.py:307-322; math of
rowfuse/ops.py:248-311 (per-row mean and inverse rms cached, centred variance,
deterministic two-stage dgamma / dbeta).  Computes in fp32, stores in the input dtype,
as Liger does.
"""

from __future__ import annotations

import torch
import torch.nn as nn

from . import errors
from ._utils import check, device_guard, dtype_code, lib, ptr, require_cuda, stream_of, workspace


@device_guard
def layer_norm_forward(X, W, B, eps):
    require_cuda(X, W, B)
    shape = X.shape
    X2 = X.reshape(-1, shape[-1]).contiguous()
    rows, cols = X2.shape
    if W.shape != (cols,) or (B is not None and B.shape != (cols,)):
        raise errors.ShapeMismatch("Incompatible hidden size dimension between input tensor and weight / bias")
    Wc = W.contiguous().to(X2.dtype)
    Bc = B.contiguous().to(X2.dtype) if B is not None else None
    Y = torch.empty_like(X2)
    mean = torch.empty(rows, dtype=torch.float32, device=X2.device)
    rstd = torch.empty(rows, dtype=torch.float32, device=X2.device)
    check(lib().lk_layernorm_fwd(ptr(X2), ptr(Wc), ptr(Bc), ptr(Y), ptr(mean), ptr(rstd), rows, cols, float(eps),
                                 dtype_code(X2), stream_of(X2)))
    return Y.view(shape), X2, mean, rstd


@device_guard
def layer_norm_backward(dY, X2, W, B, mean, rstd):
    shape = dY.shape
    dY2 = dY.reshape(-1, shape[-1]).contiguous()
    rows, cols = dY2.shape
    Wc = W.contiguous().to(X2.dtype)
    dX = torch.empty_like(dY2)
    dW = torch.empty(cols, dtype=X2.dtype, device=X2.device)
    dB = torch.empty(cols, dtype=X2.dtype, device=X2.device) if B is not None else None
    L = lib()
    ws = workspace(L.lk_layernorm_bwd_workspace_bytes(rows, cols), dY2.device)
    check(L.lk_layernorm_bwd(ptr(dY2), ptr(X2), ptr(Wc), ptr(mean), ptr(rstd), ptr(dX), ptr(dW), ptr(dB), rows,
                             cols, dtype_code(dY2), ptr(ws), ws.numel(), stream_of(dY2)))
    return dX.view(shape), dW.to(W.dtype), (dB.to(B.dtype) if dB is not None else None)


class LigerLayerNormFunction(torch.autograd.Function):
    """forward(X, W, B, eps) (LK/ops/layer_norm.py:307-322)."""

    @staticmethod
    def forward(ctx, X, W, B, eps):
        Y, X2, mean, rstd = layer_norm_forward(X, W, B, eps)
        ctx.has_b = B is not None
        ctx.save_for_backward(X2, W, B if B is not None else W, mean, rstd)
        return Y

    @staticmethod
    def backward(ctx, dY):
        X2, W, B, mean, rstd = ctx.saved_tensors
        dX, dW, dB = layer_norm_backward(dY, X2, W, B if ctx.has_b else None, mean, rstd)
        return dX, dW, dB, None


class LigerLayerNorm(nn.Module):
    """Drop-in for LK/transformers/layer_norm.py:7-25."""

    def __init__(self, hidden_size, eps=1e-6, bias=False, init_fn="ones"):
        super().__init__()
        assert init_fn in ["ones", "zeros"], f"init_fn must be either 'ones' or 'zeros', got {init_fn}"
        self.hidden_size = hidden_size
        self.eps = eps
        self.weight = nn.Parameter(torch.ones(hidden_size) if init_fn == "ones" else torch.zeros(hidden_size))
        self.bias = nn.Parameter(torch.randn(hidden_size) if bias else torch.zeros(hidden_size))
        self.variance_epsilon = eps

    def forward(self, hidden_states):
        return LigerLayerNormFunction.apply(hidden_states, self.weight, self.bias, self.variance_epsilon)

    def extra_repr(self):
        return f"{self.hidden_size}, eps={self.eps}"


def liger_layer_norm(X, W, B, eps):
    """Functional form (LK/transformers/functional.py:282-283)."""
    return LigerLayerNormFunction.apply(X, W, B, eps)
