"""Model-level training step on one B200: a Llama-3-8B-shaped decoder (HF transformers) run
stock, patched with upstream Liger-Kernel 0.8.0, and patched with this library.

It measures the drop-in at the user's level. Only the patched modules differ between the
three runs: RMSNorm, RoPE, SwiGLU MLP, and the fused linear cross entropy head. Attention
(SDPA), the projections and embeddings are identical. Each implementation runs in its own
process, because the patches are module-level.

One step is a forward with labels plus backward (no optimizer) over batch x seq tokens of
random ids. Timing uses CUDA events over `--steps` steps after `--warmup`, with inputs
resident. Peak memory is the allocator peak during one step. This is not a bench.py number.

    python scripts/model_step_bench.py [--layers 2] [--batch 4] [--seq 2048] [--impl all|hf|liger|b200]
"""

import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def run_one(impl, args):
    sys.path.insert(0, str(ROOT))
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    torch.manual_seed(0)
    dev = torch.device("cuda")
    cfg = LlamaConfig(hidden_size=4096, intermediate_size=14336, num_attention_heads=32, num_key_value_heads=8,
                      head_dim=128, vocab_size=128256, num_hidden_layers=args.layers, rope_theta=500000.0,
                      max_position_embeddings=8192, rms_norm_eps=1e-5, tie_word_embeddings=False)
    cfg._attn_implementation = "sdpa"
    model = LlamaForCausalLM(cfg).to(device=dev, dtype=torch.bfloat16).train()
    if impl == "liger":
        import torch.distributed.tensor  # noqa: F401  (liger_kernel checks DTensor)
        from liger_kernel.transformers import apply_liger_kernel_to_llama as up_apply

        up_apply(model=model)
    elif impl == "b200":
        import paper_2410_10989_b200 as lk

        lk.apply_liger_kernel_to_llama(model=model)
    g = torch.Generator(device=dev).manual_seed(1)
    ids = torch.randint(0, cfg.vocab_size, (args.batch, args.seq), device=dev, generator=g)
    labels = ids.clone()
    labels[:, : args.seq // 10] = -100

    def step():
        out = model(input_ids=ids, labels=labels)
        out.loss.backward()
        for p in model.parameters():
            p.grad = None
        return out.loss.detach()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    base = torch.cuda.memory_allocated(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    losses = [step() for _ in range(args.steps)]
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    tokens = args.batch * args.seq
    return {"impl": impl, "layers": args.layers, "tokens_per_step": tokens, "ms_per_step": round(ms, 3),
            "tokens_per_s": round(tokens / (ms / 1e3)), "peak_extra_gb": round(
                (torch.cuda.max_memory_allocated(dev) - base) / 1e9, 3), "loss": float(losses[-1])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="all", choices=["all", "hf", "liger", "b200"])
    args = ap.parse_args()
    if args.impl != "all":
        print(json.dumps(run_one(args.impl, args)), flush=True)
        return
    rows = []
    for impl in ("hf", "liger", "b200"):
        out = subprocess.run([sys.executable, __file__, "--impl", impl, "--layers", str(args.layers), "--batch",
                              str(args.batch), "--seq", str(args.seq), "--steps", str(args.steps), "--warmup",
                              str(args.warmup)], capture_output=True, text=True, cwd=ROOT)
        lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        rec = json.loads(lines[-1]) if lines else {"impl": impl, "error": out.stderr[-400:]}
        rows.append(rec)
        print(json.dumps(rec), flush=True)
    print(json.dumps({"summary": rows}))


if __name__ == "__main__":
    main()
