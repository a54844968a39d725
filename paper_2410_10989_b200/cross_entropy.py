"""Standalone cross entropy: LigerCrossEntropyFunction / LigerCrossEntropyLoss.

Drop-in for liger_kernel.transformers.LigerCrossEntropyLoss (LK/transformers/cross_entropy.py:9-61)
and LK/ops/cross_entropy.py:409-507; the algorithm is the reference's in-place
online-softmax cross entropy (rowfuse/ops.py:502-560) extended with Liger's
ignore_index / label_smoothing / softcap / z-loss semantics.  The gradient is
computed in the forward and written into the logits buffer (the reference's
in-place contract); backward only scales by grad_output.
"""

from __future__ import annotations

from dataclasses import dataclass
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
    require_cuda,
    stream_of,
    workspace,
)


@dataclass
class CrossEntropyOutput:
    loss: torch.Tensor
    z_loss: Optional[torch.Tensor] = None
    token_accuracy: Optional[torch.Tensor] = None
    predicted_tokens: Optional[torch.Tensor] = None


def _validate(label_smoothing, reduction, softcap):
    if not (0.0 <= label_smoothing <= 1.0):
        raise ValueError(f"label_smoothing must be between 0.0 and 1.0. Got: {label_smoothing}")
    if reduction not in _capi.REDUCTIONS:
        raise ValueError(f"reduction must be one of 'mean', 'sum', or 'none'. Got: {reduction}")
    if softcap is not None and not softcap > 0:
        raise ValueError(f"softcap must greater than 0.0 or None. Got: {softcap}")


@device_guard
def cross_entropy_forward(
    _input: torch.Tensor,
    target: torch.Tensor,
    weight=None,
    ignore_index: int = -100,
    lse_square_scale: float = 0.0,
    label_smoothing: float = 0.0,
    reduction: str = "mean",
    softcap: Optional[float] = None,
    return_z_loss: bool = False,
    return_token_accuracy: bool = False,
    return_predicted_tokens: bool = False,
    compute_grad: Optional[bool] = None,
):
    """Loss (+ optional z-loss) with d(loss)/d(input) left in `_input` (mirrors LK/ops/cross_entropy.py:302-407)."""
    _validate(label_smoothing, reduction, softcap)
    require_cuda(_input, target)
    if _input.dim() != 2:
        raise errors.ShapeMismatch(f"input must be (BT, V), got {tuple(_input.shape)}")
    bt, v = _input.shape
    t = as_targets(target)
    if t.numel() != bt:
        raise errors.ShapeMismatch(f"need one target per row ({bt}), got {t.numel()}")
    if _input.stride(-1) != 1:
        _input = _input.contiguous()
    grad = _input.requires_grad if compute_grad is None else compute_grad
    dev = _input.device
    loss_rows = torch.empty(bt, dtype=torch.float32, device=dev)
    loss_sum = torch.empty((), dtype=torch.float32, device=dev)
    z_rows = torch.empty(bt, dtype=torch.float32, device=dev) if return_z_loss else None
    z_sum = torch.empty((), dtype=torch.float32, device=dev) if return_z_loss else None
    cw = None
    if weight is not None:  # Liger class weights (LK/ops/cross_entropy.py:369-378)
        if weight.shape != (v,) or not torch.is_floating_point(weight):
            raise errors.ShapeMismatch(f"weight must be a floating tensor of size V={v}, got {tuple(weight.shape)}")
        cw = weight.detach().to(device=dev, dtype=torch.float32).contiguous()
    correct = torch.empty(bt, dtype=torch.float32, device=dev) if return_token_accuracy else None
    pred = torch.empty(bt, dtype=torch.int64, device=dev) if return_predicted_tokens else None
    L = lib()
    ws = workspace(L.lk_cross_entropy_workspace_bytes(bt), dev)
    staged = count_and_stage_targets(t, v, int(ignore_index))  # host check waits for this count only
    check(
        L.lk_cross_entropy_fwd_ex(
            _input.data_ptr(), _input.stride(0) if bt > 0 else v, ptr(t), bt, v, dtype_code(_input),
            int(ignore_index), float(label_smoothing), float(lse_square_scale),
            float(softcap) if softcap is not None else 0.0, _capi.REDUCTIONS[reduction], int(bool(grad)),
            loss_rows.data_ptr(), loss_sum.data_ptr(), ptr(z_rows), ptr(z_sum), ptr(correct), ptr(pred), ptr(cw),
            ws.data_ptr(), ws.numel(), stream_of(_input),
        )
    )
    counts = ws[:16].view(torch.int64)  # (n_valid, n_out_of_range) written by the kernel
    raise_if_staged_out_of_range(staged, v)
    if reduction == "none":
        loss = loss_rows.to(_input.dtype)
        z_loss = z_rows.to(_input.dtype) if return_z_loss else None
        acc = correct
    else:
        loss = loss_sum.to(_input.dtype)
        z_loss = z_sum.to(_input.dtype) if return_z_loss else None
        # mean over the non-ignored tokens for both 'mean' and 'sum' (LK/ops/cross_entropy.py:419-420)
        acc = correct.sum() / counts[0].clamp(min=1) if return_token_accuracy else None
    return loss, z_loss, acc, pred, _input


@device_guard
def cross_entropy_backward(_input: torch.Tensor, grad_output: torch.Tensor) -> torch.Tensor:
    """Scale the stored gradient by grad_output in place (LK/ops/cross_entropy.py:410-440)."""
    L = lib()
    bt, v = _input.shape
    if grad_output.ndim > 0:
        g = grad_output.reshape(-1).contiguous()
        check(L.lk_scale_rows(_input.data_ptr(), bt, v, _input.stride(0), dtype_code(_input), g.data_ptr(),
                              dtype_code(g), stream_of(_input)))
    else:
        g = grad_output.detach().to(torch.float32).reshape(1).contiguous()
        check(L.lk_scale_by_device_scalar(_input.data_ptr(), bt, v, _input.stride(0), dtype_code(_input),
                                          g.data_ptr(), stream_of(_input)))
    return _input


class LigerCrossEntropyFunction(torch.autograd.Function):
    """Same signature and return arity as LK/ops/cross_entropy.py:443-507."""

    @staticmethod
    def forward(
        ctx,
        _input: torch.Tensor,
        target: torch.Tensor,
        weight: Optional[torch.FloatTensor],
        ignore_index: int = -100,
        lse_square_scale: float = 0.0,
        label_smoothing: float = 0.0,
        reduction: str = "mean",
        softcap: Optional[float] = None,
        return_z_loss: bool = False,
        return_token_accuracy: bool = False,
        return_predicted_tokens: bool = False,
    ):
        input_requires_grad = _input.requires_grad
        loss, z_loss, acc, pred, grad_in = cross_entropy_forward(
            _input, target, weight, ignore_index, lse_square_scale, label_smoothing, reduction, softcap,
            return_z_loss, return_token_accuracy, return_predicted_tokens, compute_grad=input_requires_grad,
        )
        if input_requires_grad:
            ctx.save_for_backward(grad_in.detach())
        ctx.return_z_loss = return_z_loss
        return loss, z_loss, acc, pred

    @staticmethod
    def backward(ctx, grad_output, grad_output2, grad_output3, grad_output4):
        (_input,) = ctx.saved_tensors
        _input = cross_entropy_backward(_input, grad_output)
        return (_input, None, None, None, None, None, None, None, None, None, None)


class LigerCrossEntropyLoss(torch.nn.Module):
    """Drop-in for LK/transformers/cross_entropy.py:9-61."""

    def __init__(
        self,
        weight: Optional[torch.FloatTensor] = None,
        ignore_index: int = -100,
        lse_square_scale: float = 0.0,
        label_smoothing: float = 0.0,
        reduction: str = "mean",
        softcap: Optional[float] = None,
        return_z_loss: bool = False,
        return_token_accuracy: bool = False,
        return_predicted_tokens: bool = False,
    ):
        super().__init__()
        assert 0 <= label_smoothing <= 1, f"label_smoothing must be between 0.0 and 1.0. Got: {label_smoothing}"
        assert reduction in {"mean", "sum", "none"}, f"reduction must be one of 'mean', 'sum', or 'none'. Got: {reduction}"
        assert softcap is None or softcap > 0, f"softcap must greater than 0.0 or None. Got: {softcap}"
        self.weight = weight
        self.ignore_index = ignore_index
        self.lse_square_scale = lse_square_scale
        self.label_smoothing = label_smoothing
        self.reduction = reduction
        self.softcap = softcap
        self.return_z_loss = return_z_loss
        self.return_token_accuracy = return_token_accuracy
        self.return_predicted_tokens = return_predicted_tokens

    def forward(self, _input: torch.Tensor, target: torch.Tensor):
        loss, z_loss, acc, pred = LigerCrossEntropyFunction.apply(
            _input, target, self.weight, self.ignore_index, self.lse_square_scale, self.label_smoothing,
            self.reduction, self.softcap, self.return_z_loss, self.return_token_accuracy,
            self.return_predicted_tokens,
        )
        if not self.return_z_loss and not self.return_token_accuracy and not self.return_predicted_tokens:
            return loss
        return CrossEntropyOutput(loss=loss, z_loss=z_loss, token_accuracy=acc, predicted_tokens=pred)
