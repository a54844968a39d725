"""B200-native (sm_100a) Liger training hot path.

Drop-in Liger operator surface (liger_kernel 0.8.0 names and signatures) whose
forward and backward run hand-written sm_100a CUDA through the C ABI in
include/liger_b200.h.  No Triton, no multi-backend dispatch, no CPU fallback:
the ops raise ExtensionMissing / require CUDA tensors.
"""

from . import errors
from .chunking import ChunkPlan, b200_plan, plan_chunks
from .cross_entropy import CrossEntropyOutput, LigerCrossEntropyFunction, LigerCrossEntropyLoss
from .fused_linear_cross_entropy import (
    LigerFusedLinearCrossEntropyFunction,
    LigerFusedLinearCrossEntropyLoss,
    KeptRows,
    flce_plan,
    fused_linear_cross_entropy_forward,
    prepare_kept_rows,
)
from .layer_norm import LigerLayerNorm, LigerLayerNormFunction, liger_layer_norm
from .rms_norm import LigerRMSNorm, LigerRMSNormFunction
from .rope import LigerRopeFunction, liger_rotary_pos_emb
from .swiglu import (
    LigerGEGLUMLP,
    LigerGELUMulFunction,
    LigerSiLUMulFunction,
    LigerSwiGLUMLP,
    liger_geglu,
    liger_swiglu,
)

__version__ = "0.1.0"


def __getattr__(name):
    """apply_liger_kernel_to_* live in .monkey_patch (imports transformers lazily)."""
    if name.startswith("apply_liger_kernel_to_") or name in ("_apply_liger_kernel", "_apply_liger_kernel_to_instance"):
        from . import monkey_patch

        return getattr(monkey_patch, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


def liger_cross_entropy(input, target, weight=None, size_average=None, ignore_index=-100, reduce=None,
                        reduction="mean", label_smoothing=0.0, lse_square_scale=0.0, softcap=None,
                        return_z_loss=False, return_token_accuracy=False, return_predicted_tokens=False):
    """Functional form (LK/transformers/functional.py:41-77)."""
    loss, z_loss, acc, pred = LigerCrossEntropyFunction.apply(input, target, weight, ignore_index, lse_square_scale,
                                                              label_smoothing, reduction, softcap, return_z_loss,
                                                              return_token_accuracy, return_predicted_tokens)
    if not return_z_loss and not return_token_accuracy and not return_predicted_tokens:
        return loss
    return CrossEntropyOutput(loss=loss, z_loss=z_loss, token_accuracy=acc, predicted_tokens=pred)


def liger_fused_linear_cross_entropy(input, weight, target, bias=None, ce_weight=None, ignore_index=-100,
                                     lse_square_scale=0.0, label_smoothing=0.0, reduction="mean", softcap=None,
                                     return_z_loss=False, accum_dtype=None, use_token_scaling=False,
                                     return_token_accuracy=False, return_predicted_tokens=False):
    """Functional form (LK/transformers/functional.py:80-120)."""
    loss, z_loss, acc, pred = LigerFusedLinearCrossEntropyFunction.apply(
        input, weight, target, bias, ce_weight, ignore_index, lse_square_scale, label_smoothing, reduction,
        softcap, return_z_loss, accum_dtype, use_token_scaling, return_token_accuracy, return_predicted_tokens)
    if not return_z_loss and not return_token_accuracy and not return_predicted_tokens:
        return loss
    return CrossEntropyOutput(loss=loss, z_loss=z_loss, token_accuracy=acc, predicted_tokens=pred)


def liger_rms_norm(X, W, eps, offset=0.0, casting_mode="llama", in_place=True):
    return LigerRMSNormFunction.apply(X, W, eps, offset, casting_mode, in_place)


__all__ = [
    "errors", "ChunkPlan", "plan_chunks", "b200_plan", "flce_plan",
    "CrossEntropyOutput", "LigerCrossEntropyFunction", "LigerCrossEntropyLoss",
    "LigerFusedLinearCrossEntropyFunction", "LigerFusedLinearCrossEntropyLoss",
    "fused_linear_cross_entropy_forward", "prepare_kept_rows", "KeptRows",
    "LigerRMSNorm", "LigerRMSNormFunction", "LigerLayerNorm", "LigerLayerNormFunction", "liger_layer_norm", "LigerRopeFunction", "liger_rotary_pos_emb",
    "LigerSiLUMulFunction", "LigerGELUMulFunction", "LigerSwiGLUMLP", "LigerGEGLUMLP",
    "liger_swiglu", "liger_geglu", "liger_cross_entropy", "liger_fused_linear_cross_entropy", "liger_rms_norm",
]
