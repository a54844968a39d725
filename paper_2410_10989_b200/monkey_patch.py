"""HuggingFace model patching: apply_liger_kernel_to_<model>.

Drop-in for LK/transformers/monkey_patch.py (liger_kernel 0.8.0): the same entry points,
keyword arguments and patch targets, routing the decoder's RMSNorm, RoPE and GLU MLP and
the causal-LM loss through this package's sm_100a kernels.

  * class-level (before the model is built): the modeling module's RMSNorm / MLP classes
    and its ``apply_rotary_pos_emb`` are swapped, and ``<Model>ForCausalLM.forward``
    becomes :func:`lce_forward` (LK/transformers/monkey_patch.py:221-285);
  * instance-level (``model=...``): the already-built norm and MLP modules get their
    ``forward`` rebound in place, keeping their parameters (monkey_patch.py:63-143).

:func:`lce_forward` follows LK/transformers/model/llama.py:24-160: in training with labels
(``skip_logits``), the final hidden states go straight into the fused linear cross entropy
(the chunked tcgen05 head; logits never materialised), with the model's
``final_logit_softcapping`` as ``softcap`` (Gemma-2); otherwise logits are materialised
and the stock ``loss_function`` runs.  Families covered: the two north-star heads (Llama,
Gemma-2) and the decoders that share their blocks (Mistral, Qwen2, Qwen3, Gemma).
"""

from __future__ import annotations

import inspect
import logging
from dataclasses import dataclass
from functools import partial
from types import MethodType
from typing import Optional

import torch
import torch.nn as nn

from .cross_entropy import CrossEntropyOutput
from .rms_norm import LigerRMSNorm
from .rope import liger_rotary_pos_emb
from .swiglu import LigerGEGLUMLP, LigerSwiGLUMLP

logger = logging.getLogger(__name__)

try:  # transformers is optional for the kernels, required for patching
    from transformers.modeling_outputs import CausalLMOutputWithPast
except ImportError:  # pragma: no cover
    CausalLMOutputWithPast = object


class LigerRMSNormForGemma(LigerRMSNorm):
    """GemmaRMSNorm: (1 + w) offset, fp32 'gemma' casting, zero init (LK/transformers/rms_norm.py:49-57)."""

    def __init__(self, hidden_size, eps=1e-6, offset=1.0, casting_mode="gemma", init_fn="zeros", in_place=True,
                 row_mode=None):
        super().__init__(hidden_size, eps, offset, casting_mode, init_fn, in_place, row_mode)


class LigerRMSNormForGemma2(LigerRMSNorm):
    """Gemma2RMSNorm; not in place, the residual reads the input again (LK/transformers/rms_norm.py:59-64)."""

    def __init__(self, hidden_size, eps=1e-6, offset=1.0, casting_mode="gemma", init_fn="zeros", in_place=False,
                 row_mode=None):
        super().__init__(hidden_size, eps, offset, casting_mode, init_fn, in_place, row_mode)


@dataclass
class LigerCausalLMOutputWithPast(CausalLMOutputWithPast):
    """CausalLMOutputWithPast plus the FLCE side outputs (LK/transformers/model/output_classes.py)."""

    token_accuracy: Optional[torch.Tensor] = None
    predicted_tokens: Optional[torch.Tensor] = None


def unpack_cross_entropy_result(result):
    """(loss, z_loss, token_accuracy, predicted_tokens) (LK/transformers/model/loss_utils.py:14-29)."""
    if isinstance(result, CrossEntropyOutput):
        return result.loss, result.z_loss, result.token_accuracy, result.predicted_tokens
    if isinstance(result, tuple):
        pad = tuple(result) + (None,) * (4 - len(result))
        return pad[0], pad[1], pad[2], pad[3]
    return result, None, None, None


def LigerForCausalLMLoss(hidden_states, lm_head_weight, labels, hidden_size: int, num_items_in_batch=None,
                         ignore_index: int = -100, shift_labels=None, final_logit_softcapping=None,
                         return_token_accuracy: bool = False, return_predicted_tokens: bool = False,
                         lm_head_bias=None, **kwargs):
    """Shifted next-token loss through the fused head (LK/transformers/model/loss_utils.py:32-100).

    ``num_items_in_batch`` (gradient accumulation) switches to a SUM reduction divided by it.
    """
    from . import liger_fused_linear_cross_entropy

    allowed = inspect.signature(liger_fused_linear_cross_entropy).parameters
    kwargs = {k: v for k, v in kwargs.items() if k in allowed}
    if shift_labels is None:
        labels = nn.functional.pad(labels, (0, 1), value=ignore_index)
        shift_labels = labels[..., 1:].contiguous()
    hidden_states = hidden_states.reshape(-1, hidden_size)
    shift_labels = shift_labels.reshape(-1).to(hidden_states.device)
    reduction = "sum" if num_items_in_batch is not None else "mean"
    result = liger_fused_linear_cross_entropy(
        hidden_states, lm_head_weight, shift_labels, bias=lm_head_bias, ignore_index=ignore_index,
        reduction=reduction, softcap=final_logit_softcapping, return_token_accuracy=return_token_accuracy,
        return_predicted_tokens=return_predicted_tokens, **kwargs)
    loss, _, acc, pred = unpack_cross_entropy_result(result)
    if reduction == "sum":
        loss = loss / num_items_in_batch
    if return_token_accuracy or return_predicted_tokens:
        return CrossEntropyOutput(loss=loss, token_accuracy=acc, predicted_tokens=pred)
    return loss


def lce_forward(self, input_ids=None, attention_mask=None, position_ids=None, past_key_values=None,
                inputs_embeds=None, labels=None, use_cache=None, logits_to_keep=0, skip_logits=None,
                return_dict=None, **kwargs):
    """<Model>ForCausalLM.forward with the fused head (LK/transformers/model/llama.py:24-160)."""
    if getattr(self.config, "pretraining_tp", 1) > 1:
        raise NotImplementedError("pretraining_tp > 1 is not supported")
    shift_labels = kwargs.pop("shift_labels", None)
    head_loss = skip_logits if skip_logits is not None else (
        self.training and (labels is not None or shift_labels is not None))
    if head_loss and (labels is not None or shift_labels is not None):
        # the fused head skips ignore_index rows; its row compaction is enqueued here, before
        # the decoder runs, so the head later sizes its chunk loop from a count the GPU produced
        # long before instead of waiting for the whole forward (prepare_kept_rows)
        if shift_labels is None:
            shift_labels = nn.functional.pad(labels, (0, 1), value=kwargs.get("ignore_index", -100))[..., 1:]
            shift_labels = shift_labels.contiguous()
        if shift_labels.is_cuda:
            from .fused_linear_cross_entropy import prepare_kept_rows

            prepare_kept_rows(shift_labels.reshape(-1), ignore_index=kwargs.get("ignore_index", -100))
    outputs = self.model(input_ids=input_ids, attention_mask=attention_mask, position_ids=position_ids,
                         past_key_values=past_key_values, inputs_embeds=inputs_embeds, use_cache=use_cache, **kwargs)
    hidden_states = outputs[0]
    slice_indices = slice(-logits_to_keep, None) if isinstance(logits_to_keep, int) else logits_to_keep
    kept = hidden_states[:, slice_indices, :]
    softcap = getattr(self.config, "final_logit_softcapping", None)

    if skip_logits and labels is None and shift_labels is None:
        raise ValueError("skip_logits is True, but labels and shift_labels are None")
    if skip_logits is None:
        skip_logits = self.training and (labels is not None or shift_labels is not None)

    logits = loss = acc = pred = None
    if skip_logits:
        result = LigerForCausalLMLoss(kept, self.lm_head.weight, labels, self.config.hidden_size,
                                      shift_labels=shift_labels, final_logit_softcapping=softcap,
                                      lm_head_bias=getattr(self.lm_head, "bias", None), **kwargs)
        loss, _, acc, pred = unpack_cross_entropy_result(result)
    else:
        logits = self.lm_head(kept)
        if softcap is not None:
            logits = torch.tanh(logits / softcap) * softcap
        if labels is not None or shift_labels is not None:
            loss = self.loss_function(logits=logits, labels=labels, shift_labels=shift_labels,
                                      vocab_size=self.config.vocab_size, **kwargs)

    if return_dict is False:
        out = (logits,) + tuple(outputs[1:])
        out = ((loss,) + out) if loss is not None else out
        out = out + (acc,) if acc is not None else out
        return out + (pred,) if pred is not None else out
    return LigerCausalLMOutputWithPast(loss=loss, logits=logits, past_key_values=outputs.past_key_values,
                                       hidden_states=outputs.hidden_states, attentions=outputs.attentions,
                                       token_accuracy=acc, predicted_tokens=pred)


def _bind_method_to_module(module, method_name, new_method):
    module.__dict__[method_name] = new_method.__get__(module, module.__class__)


def _patch_rms_norm_module(module, offset=0.0, eps=1e-6, casting_mode="llama", in_place=True, row_mode=None):
    """Rebind a built HF RMSNorm to LigerRMSNorm.forward, keeping its weight (monkey_patch.py:68-115)."""
    module.offset = offset
    module.casting_mode = casting_mode
    module.variance_epsilon = getattr(module, "variance_epsilon", None) or getattr(module, "eps", None) or eps
    module.in_place = in_place
    module.row_mode = row_mode
    _bind_method_to_module(module, "forward", LigerRMSNorm.forward)
    _bind_method_to_module(module, "extra_repr", LigerRMSNorm.extra_repr)
    _bind_method_to_module(module, "_get_name", lambda self: LigerRMSNorm.__name__)


def _patch_swiglu_module(module, liger_module=LigerSwiGLUMLP):
    _bind_method_to_module(module, "forward", liger_module.forward)
    _bind_method_to_module(module, "_get_name", lambda self: liger_module.__name__)


def _patch_geglu_module(module):
    _patch_swiglu_module(module, LigerGEGLUMLP)


def _check_loss_flags(cross_entropy, fused_linear_cross_entropy):
    assert not (cross_entropy and fused_linear_cross_entropy), (
        "cross_entropy and fused_linear_cross_entropy cannot both be True.")


def _patch_cross_entropy():
    """The stock HF loss_function calls nn.functional.cross_entropy (transformers/loss/loss_utils.py)."""
    from transformers.loss.loss_utils import nn as loss_nn

    from . import liger_cross_entropy

    loss_nn.functional.cross_entropy = liger_cross_entropy


def _apply_decoder(module, prefix, *, rope, cross_entropy, fused_linear_cross_entropy, rms_norm, mlp, mlp_cls,
                   norm_cls, norm_patch, norm_names, model, qk_norm=False):
    """Shared body of the per-family entry points below."""
    _check_loss_flags(cross_entropy, fused_linear_cross_entropy)
    if rope:
        module.apply_rotary_pos_emb = liger_rotary_pos_emb
    if rms_norm:
        setattr(module, f"{prefix}RMSNorm", norm_cls)
    if mlp:
        setattr(module, f"{prefix}MLP", mlp_cls)
    if cross_entropy:
        _patch_cross_entropy()
    if fused_linear_cross_entropy:
        if model is not None:
            model.forward = MethodType(lce_forward, model)
        else:
            getattr(module, f"{prefix}ForCausalLM").forward = lce_forward
    if model is None:
        return
    base = getattr(model, model.base_model_prefix, model)
    if rms_norm:
        norm_patch(base.norm)
    for layer in base.layers:
        if mlp:
            _patch_swiglu_module(layer.mlp, mlp_cls)
        if rms_norm:
            for name in norm_names:
                norm_patch(getattr(layer, name))
            if qk_norm:
                norm_patch(layer.self_attn.q_norm)
                norm_patch(layer.self_attn.k_norm)


_LLAMA_NORMS = ("input_layernorm", "post_attention_layernorm")


def apply_liger_kernel_to_llama(rope=True, cross_entropy=False, fused_linear_cross_entropy=True, rms_norm=True,
                                swiglu=True, model=None) -> None:
    """Llama 2/3 (LK/transformers/monkey_patch.py:221-285)."""
    from transformers.models.llama import modeling_llama

    _apply_decoder(modeling_llama, "Llama", rope=rope, cross_entropy=cross_entropy,
                   fused_linear_cross_entropy=fused_linear_cross_entropy, rms_norm=rms_norm, mlp=swiglu,
                   mlp_cls=LigerSwiGLUMLP, norm_cls=LigerRMSNorm, norm_patch=_patch_rms_norm_module,
                   norm_names=_LLAMA_NORMS, model=model)


def apply_liger_kernel_to_mistral(rope=True, cross_entropy=False, fused_linear_cross_entropy=True, rms_norm=True,
                                  swiglu=True, model=None) -> None:
    """Mistral (LK/transformers/monkey_patch.py apply_liger_kernel_to_mistral)."""
    from transformers.models.mistral import modeling_mistral

    _apply_decoder(modeling_mistral, "Mistral", rope=rope, cross_entropy=cross_entropy,
                   fused_linear_cross_entropy=fused_linear_cross_entropy, rms_norm=rms_norm, mlp=swiglu,
                   mlp_cls=LigerSwiGLUMLP, norm_cls=LigerRMSNorm, norm_patch=_patch_rms_norm_module,
                   norm_names=_LLAMA_NORMS, model=model)


def apply_liger_kernel_to_qwen2(rope=True, cross_entropy=False, fused_linear_cross_entropy=True, rms_norm=True,
                                swiglu=True, model=None) -> None:
    """Qwen2 (LK/transformers/monkey_patch.py apply_liger_kernel_to_qwen2)."""
    from transformers.models.qwen2 import modeling_qwen2

    _apply_decoder(modeling_qwen2, "Qwen2", rope=rope, cross_entropy=cross_entropy,
                   fused_linear_cross_entropy=fused_linear_cross_entropy, rms_norm=rms_norm, mlp=swiglu,
                   mlp_cls=LigerSwiGLUMLP, norm_cls=LigerRMSNorm, norm_patch=_patch_rms_norm_module,
                   norm_names=_LLAMA_NORMS, model=model)


def apply_liger_kernel_to_qwen3(rope=True, cross_entropy=False, fused_linear_cross_entropy=True, rms_norm=True,
                                swiglu=True, model=None) -> None:
    """Qwen3: also the per-head q_norm / k_norm (LK/transformers/monkey_patch.py apply_liger_kernel_to_qwen3)."""
    from transformers.models.qwen3 import modeling_qwen3

    _apply_decoder(modeling_qwen3, "Qwen3", rope=rope, cross_entropy=cross_entropy,
                   fused_linear_cross_entropy=fused_linear_cross_entropy, rms_norm=rms_norm, mlp=swiglu,
                   mlp_cls=LigerSwiGLUMLP, norm_cls=LigerRMSNorm, norm_patch=_patch_rms_norm_module,
                   norm_names=_LLAMA_NORMS, model=model, qk_norm=True)


def apply_liger_kernel_to_gemma(rope=True, cross_entropy=False, fused_linear_cross_entropy=True, rms_norm=True,
                                geglu=True, model=None) -> None:
    """Gemma 1 / 1.1 (LK/transformers/monkey_patch.py:920-990)."""
    from transformers.models.gemma import modeling_gemma

    _apply_decoder(modeling_gemma, "Gemma", rope=rope, cross_entropy=cross_entropy,
                   fused_linear_cross_entropy=fused_linear_cross_entropy, rms_norm=rms_norm, mlp=geglu,
                   mlp_cls=LigerGEGLUMLP, norm_cls=LigerRMSNormForGemma,
                   norm_patch=partial(_patch_rms_norm_module, offset=1.0, casting_mode="gemma"),
                   norm_names=_LLAMA_NORMS, model=model)


def apply_liger_kernel_to_gemma2(rope=True, cross_entropy=False, fused_linear_cross_entropy=True, rms_norm=True,
                                 geglu=True, model=None) -> None:
    """Gemma 2: four norms per layer, final-logit softcap into the FLCE (monkey_patch.py:993-1061)."""
    from transformers.models.gemma2 import modeling_gemma2

    _apply_decoder(modeling_gemma2, "Gemma2", rope=rope, cross_entropy=cross_entropy,
                   fused_linear_cross_entropy=fused_linear_cross_entropy, rms_norm=rms_norm, mlp=geglu,
                   mlp_cls=LigerGEGLUMLP, norm_cls=LigerRMSNormForGemma2,
                   norm_patch=partial(_patch_rms_norm_module, offset=1.0, casting_mode="gemma", in_place=False),
                   norm_names=_LLAMA_NORMS + ("pre_feedforward_layernorm", "post_feedforward_layernorm"),
                   model=model)


MODEL_TYPE_TO_APPLY_LIGER_FN = {
    "llama": apply_liger_kernel_to_llama,
    "mistral": apply_liger_kernel_to_mistral,
    "qwen2": apply_liger_kernel_to_qwen2,
    "qwen3": apply_liger_kernel_to_qwen3,
    "gemma": apply_liger_kernel_to_gemma,
    "gemma2": apply_liger_kernel_to_gemma2,
}


def _filtered(fn, kwargs):
    params = inspect.signature(fn).parameters
    return {k: v for k, v in kwargs.items() if k in params}


def _apply_liger_kernel(model_type: str, **kwargs) -> None:
    """Class-level patch by config.model_type (LK/transformers/monkey_patch.py:3411-3443)."""
    fn = MODEL_TYPE_TO_APPLY_LIGER_FN.get(model_type) if model_type else None
    if fn is None:
        logger.info("no Liger kernels for model type %r", model_type)
        return
    fn(**_filtered(fn, kwargs))


def _apply_liger_kernel_to_instance(model, **kwargs) -> None:
    """Instance-level patch of a built model (LK/transformers/monkey_patch.py:3446-3473)."""
    model_type = getattr(getattr(model, "config", None), "model_type", None)
    fn = MODEL_TYPE_TO_APPLY_LIGER_FN.get(model_type) if model_type else None
    if fn is None:
        logger.info("no Liger kernels for model type %r", model_type)
        return
    fn(model=model, **_filtered(fn, kwargs))
