"""SwiGLU / GeGLU: LigerSiLUMulFunction, LigerGELUMulFunction, LigerSwiGLUMLP, LigerGEGLUMLP.

Drop-ins for LK/ops/swiglu.py:110-160, LK/ops/geglu.py:112-140 and the MLP
modules of LK/transformers/swiglu.py:8-21 / geglu.py:6-24.  Elementwise math of
rowfuse/ops.py:389-482; the backward recomputes the activation and writes da, db
into the saved a, b buffers in place, as Liger does.
"""

from __future__ import annotations

import torch
import torch.nn as nn

from . import errors
from ._utils import check, device_guard, dtype_code, lib, require_cuda, stream_of


@device_guard
def _fwd(fn_name, a, b, *extra):
    require_cuda(a, b)
    if a.shape != b.shape or a.dtype != b.dtype:
        raise errors.ShapeMismatch("gate and up halves must match in shape and dtype (rowfuse/ops.py:99-106)")
    # fresh view objects (same storage): the backward writes da/db into them and returns them,
    # and autograd can then take them as leaf .grad without a defensive copy (as Liger's
    # a.view(-1, n) does)
    a = a.contiguous().view(a.shape)
    b = b.contiguous().view(b.shape)
    c = torch.empty_like(a)
    check(getattr(lib(), fn_name)(a.data_ptr(), b.data_ptr(), c.data_ptr(), a.numel(), *extra, dtype_code(a),
                                  stream_of(a)))
    return a, b, c


@device_guard
def _bwd(fn_name, a, b, dc, *extra):
    dc = dc.contiguous()
    check(getattr(lib(), fn_name)(dc.data_ptr(), a.data_ptr(), b.data_ptr(), a.numel(), *extra, dtype_code(a),
                                  stream_of(a)))
    return a, b


def swiglu_forward(a, b, gate_multiplier: float = 1.0):
    """c = silu(gate_multiplier * a) * b (LK/ops/swiglu.py:65-86)."""
    return _fwd("lk_swiglu_fwd_ex", a, b, float(gate_multiplier))


def swiglu_backward(a, b, dc, gate_multiplier: float = 1.0):
    return _bwd("lk_swiglu_bwd_ex", a, b, dc, float(gate_multiplier))


def geglu_forward(a, b):
    return _fwd("lk_geglu_fwd", a, b)


def geglu_backward(a, b, dc):
    return _bwd("lk_geglu_bwd", a, b, dc)


class LigerSiLUMulFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b, gate_multiplier: float = 1.0, down_multiplier: float = 1.0):
        """LK/ops/swiglu.py:110-160: c = silu(gate_multiplier * a) * b * down_multiplier."""
        a, b, c = swiglu_forward(a, b, gate_multiplier)
        if float(down_multiplier) != 1.0:
            c = c * down_multiplier
        ctx.gate_multiplier = float(gate_multiplier)
        ctx.down_multiplier = float(down_multiplier)
        ctx.save_for_backward(a, b)
        return c

    @staticmethod
    def backward(ctx, dc):
        a, b = ctx.saved_tensors
        if ctx.down_multiplier != 1.0:
            dc = dc * ctx.down_multiplier
        a, b = swiglu_backward(a, b, dc, ctx.gate_multiplier)
        return a, b, None, None


class LigerGELUMulFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b):
        a, b, c = geglu_forward(a, b)
        ctx.save_for_backward(a, b)
        return c

    @staticmethod
    def backward(ctx, dc):
        a, b = ctx.saved_tensors
        a, b = geglu_backward(a, b, dc)
        return a, b


class LigerSwiGLUMLP(nn.Module):
    """down(silu(gate(x)) * up(x)) — LK/transformers/swiglu.py:8-21."""

    def __init__(self, config):
        super().__init__()
        self.config = config
        self.hidden_size = config.hidden_size
        self.intermediate_size = config.intermediate_size
        self.gate_proj = nn.Linear(self.hidden_size, self.intermediate_size, bias=False)
        self.up_proj = nn.Linear(self.hidden_size, self.intermediate_size, bias=False)
        self.down_proj = nn.Linear(self.intermediate_size, self.hidden_size, bias=False)
        if config.hidden_act not in ["silu", "swish"]:
            raise ValueError(f"Activation function {config.hidden_act} not supported.")

    def forward(self, x):
        return self.down_proj(LigerSiLUMulFunction.apply(self.gate_proj(x), self.up_proj(x)))


class LigerGEGLUMLP(nn.Module):
    """down(gelu_tanh(gate(x)) * up(x)) — LK/transformers/geglu.py:6-24."""

    def __init__(self, config):
        super().__init__()
        self.config = config
        self.hidden_size = config.hidden_size
        self.intermediate_size = config.intermediate_size
        self.gate_proj = nn.Linear(self.hidden_size, self.intermediate_size, bias=False)
        self.up_proj = nn.Linear(self.hidden_size, self.intermediate_size, bias=False)
        self.down_proj = nn.Linear(self.intermediate_size, self.hidden_size, bias=False)

    def forward(self, x):
        return self.down_proj(LigerGELUMulFunction.apply(self.gate_proj(x), self.up_proj(x)))


def liger_swiglu(a, b):
    return LigerSiLUMulFunction.apply(a, b)


def liger_geglu(a, b):
    return LigerGELUMulFunction.apply(a, b)
