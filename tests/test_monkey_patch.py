"""HF model patching (paper_2410_10989_b200.monkey_patch), modelled on Liger's
test/transformers/test_monkey_patch.py (instance and class patching) and
test/convergence (patched vs stock model, same weights, same batch).

CPU: which modules get patched, kwargs filtering, the class-level swap.
GPU: tiny Llama / Mistral / Qwen3 / Gemma / Gemma-2 decoders, patched copy vs stock
model: loss, every parameter gradient and the eval-mode logits.
"""

import contextlib
import copy
import importlib

import pytest
import torch

transformers = pytest.importorskip("transformers")

from paper_2410_10989_b200 import LigerGEGLUMLP, LigerRMSNorm, LigerSwiGLUMLP  # noqa: E402
from paper_2410_10989_b200 import monkey_patch as mp  # noqa: E402

FAMILIES = {
    # model_type: (module, prefix, config class, causal-LM class, extra config kwargs)
    "llama": ("llama", "Llama", "LlamaConfig", "LlamaForCausalLM", {}),
    "mistral": ("mistral", "Mistral", "MistralConfig", "MistralForCausalLM", {}),
    "qwen3": ("qwen3", "Qwen3", "Qwen3Config", "Qwen3ForCausalLM", {"head_dim": 64}),
    "gemma": ("gemma", "Gemma", "GemmaConfig", "GemmaForCausalLM", {"head_dim": 64}),
    "gemma2": ("gemma2", "Gemma2", "Gemma2Config", "Gemma2ForCausalLM",
               {"head_dim": 64, "final_logit_softcapping": 30.0, "attn_logit_softcapping": 50.0}),
}


def _modeling(mt):
    return importlib.import_module(f"transformers.models.{FAMILIES[mt][0]}.modeling_{FAMILIES[mt][0]}")


@contextlib.contextmanager
def restored(mt):
    """Undo the module-level swaps the patch functions make."""
    from transformers.loss.loss_utils import nn as loss_nn

    mod = _modeling(mt)
    prefix = FAMILIES[mt][1]
    names = ("apply_rotary_pos_emb", f"{prefix}RMSNorm", f"{prefix}MLP")
    saved = {n: getattr(mod, n) for n in names}
    lm_cls = getattr(mod, f"{prefix}ForCausalLM")
    fwd = lm_cls.__dict__["forward"]
    ce = loss_nn.functional.cross_entropy
    try:
        yield mod
    finally:
        for n, v in saved.items():
            setattr(mod, n, v)
        lm_cls.forward = fwd
        loss_nn.functional.cross_entropy = ce


def _tiny(mt, dtype=torch.float32, device="cpu"):
    _, _, cfg_name, lm_name, extra = FAMILIES[mt]
    cfg = getattr(transformers, cfg_name)(
        vocab_size=1024, hidden_size=256, intermediate_size=512, num_hidden_layers=2, num_attention_heads=4,
        num_key_value_heads=2, max_position_embeddings=256, rms_norm_eps=1e-6, attn_implementation="eager",
        **extra)
    torch.manual_seed(0)
    model = getattr(transformers, lm_name)(cfg)
    with torch.no_grad():  # non-trivial norm weights (Gemma's init to zero)
        for name, p in model.named_parameters():
            if "norm" in name:
                p.copy_(torch.rand_like(p) * 0.5 + (0.0 if mt.startswith("gemma") else 0.75))
    return model.to(device=device, dtype=dtype)


def _norms(model):
    base = model.model
    out = [base.norm]
    for layer in base.layers:
        out += [m for n, m in layer.named_modules() if n.endswith("norm")]
    return out


@pytest.mark.parametrize("mt", sorted(FAMILIES))
def test_instance_patch_binds_modules(mt):
    model = _tiny(mt)
    with restored(mt):
        mp._apply_liger_kernel_to_instance(model, swiglu=True, geglu=True, unknown_flag=1)
        assert model.forward.__func__ is mp.lce_forward
        for n in _norms(model):
            assert n.forward.__func__ is LigerRMSNorm.forward
            assert n._get_name() == "LigerRMSNorm"
            assert n.offset == (1.0 if mt.startswith("gemma") else 0.0)
            assert n.casting_mode == ("gemma" if mt.startswith("gemma") else "llama")
            assert n.variance_epsilon == 1e-6
        if mt == "gemma2":
            assert all(not n.in_place for n in _norms(model))
        if mt == "qwen3":
            assert model.model.layers[0].self_attn.q_norm.forward.__func__ is LigerRMSNorm.forward
        mlp_cls = LigerGEGLUMLP if mt.startswith("gemma") else LigerSwiGLUMLP
        for layer in model.model.layers:
            assert layer.mlp.forward.__func__ is mlp_cls.forward
        assert _modeling(mt).apply_rotary_pos_emb is mp.liger_rotary_pos_emb
    assert _modeling(mt).apply_rotary_pos_emb is not mp.liger_rotary_pos_emb


def test_class_patch_swaps_classes():
    with restored("llama") as mod:
        mp._apply_liger_kernel("llama", rms_norm=True, swiglu=True, rope=True, geglu=True)
        assert mod.LlamaRMSNorm is LigerRMSNorm and mod.LlamaMLP is LigerSwiGLUMLP
        assert mod.LlamaForCausalLM.forward is mp.lce_forward
        model = _tiny("llama")
        assert isinstance(model.model.norm, LigerRMSNorm)
        assert isinstance(model.model.layers[0].mlp, LigerSwiGLUMLP)
    with restored("gemma2") as mod:
        mp.apply_liger_kernel_to_gemma2(fused_linear_cross_entropy=False, cross_entropy=True)
        assert mod.Gemma2RMSNorm is mp.LigerRMSNormForGemma2 and mod.Gemma2MLP is LigerGEGLUMLP
        from transformers.loss.loss_utils import nn as loss_nn

        import paper_2410_10989_b200 as lk
        assert loss_nn.functional.cross_entropy is lk.liger_cross_entropy
    with pytest.raises(AssertionError):
        mp.apply_liger_kernel_to_llama(cross_entropy=True, fused_linear_cross_entropy=True)


def test_unknown_model_type_is_a_noop():
    mp._apply_liger_kernel("not_a_model")
    mp._apply_liger_kernel(None)


def test_unpack_cross_entropy_result():
    t = torch.tensor(1.0)
    assert mp.unpack_cross_entropy_result(t) == (t, None, None, None)
    assert mp.unpack_cross_entropy_result((t, 2)) == (t, 2, None, None)
    r = mp.CrossEntropyOutput(loss=t, token_accuracy=3)
    assert mp.unpack_cross_entropy_result(r) == (t, None, 3, None)


def _grad_gap(ref, fused):
    worst = 0.0
    pr = dict(ref.named_parameters())
    for name, p in fused.named_parameters():
        g, gr = p.grad.float(), pr[name].grad.float()
        worst = max(worst, float((g - gr).abs().max() / gr.abs().max().clamp_min(1e-12)))
    return worst


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
@pytest.mark.parametrize("mt", sorted(FAMILIES))
def test_patched_model_matches_stock(mt, dtype):
    """Training step with labels: fused head (no logits) vs stock; then eval logits."""
    dev = torch.device("cuda")
    ref = _tiny(mt, dtype, dev).train()
    fused = copy.deepcopy(ref)
    g = torch.Generator(device=dev).manual_seed(1)
    ids = torch.randint(0, 1024, (2, 96), device=dev, generator=g)
    labels = ids.clone()
    labels[:, :7] = -100
    with restored(mt):
        out_r = ref(input_ids=ids, labels=labels)  # before the module-level rope swap
        out_r.loss.backward()
        with torch.no_grad():
            logits_r = ref.eval()(input_ids=ids).logits.float()
        mp._apply_liger_kernel_to_instance(fused)
        out_f = fused(input_ids=ids, labels=labels)
        assert out_f.logits is None  # the fused head never materialises logits
        out_f.loss.backward()
        with torch.no_grad():
            logits_f = fused.eval()(input_ids=ids).logits.float()
    loss_tol, grad_tol = (1e-4, 2e-3) if dtype == torch.float32 else (2e-2, 6e-2)
    assert abs(out_f.loss.item() - out_r.loss.item()) <= loss_tol * abs(out_r.loss.item())
    assert _grad_gap(ref, fused) <= grad_tol
    gap = float((logits_f - logits_r).abs().max() / logits_r.abs().max())
    assert gap <= (1e-4 if dtype == torch.float32 else 3e-2)


@pytest.mark.gpu
def test_patched_llama_num_items_and_accuracy():
    """Gradient-accumulation normalisation (num_items_in_batch) and token accuracy through lce_forward."""
    dev = torch.device("cuda")
    model = _tiny("llama", torch.float32, dev).train()
    ids = torch.randint(0, 1024, (2, 64), device=dev)
    with restored("llama"):
        mp.apply_liger_kernel_to_llama(model=model)
        base = model(input_ids=ids, labels=ids).loss
        n = int((ids[:, 1:] != -100).sum())
        scaled = model(input_ids=ids, labels=ids, num_items_in_batch=2 * n).loss
        torch.testing.assert_close(scaled, base / 2, rtol=1e-5, atol=1e-6)
        out = model(input_ids=ids, labels=ids, return_token_accuracy=True)
        assert out.token_accuracy is not None and 0.0 <= float(out.token_accuracy) <= 1.0


@pytest.mark.gpu
def test_patched_llama_cross_entropy_path_matches_stock():
    """cross_entropy=True: the stock HF loss_function runs with nn.functional.cross_entropy
    swapped for the library's CE (materialised logits)."""
    dev = torch.device("cuda")
    ref = _tiny("llama", torch.float32, dev).train()
    fused = copy.deepcopy(ref)
    ids = torch.randint(0, 1024, (2, 80), device=dev)
    with restored("llama"):
        out_r = ref(input_ids=ids, labels=ids)
        out_r.loss.backward()
        mp.apply_liger_kernel_to_llama(cross_entropy=True, fused_linear_cross_entropy=False, model=fused)
        out_f = fused(input_ids=ids, labels=ids)
        assert out_f.logits is not None
        out_f.loss.backward()
    assert abs(out_f.loss.item() - out_r.loss.item()) <= 1e-4 * abs(out_r.loss.item())
    assert _grad_gap(ref, fused) <= 2e-3
