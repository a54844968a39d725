"""grad_w accumulation across chunks on the cfg2 FLCE, interleaved A/B (GPU).

    python scripts/dw_accum_probe.py [rounds]
Configs: bf16 in grad_w by TMA reduce-add in L2 (LK_PATH_DW_ACCUM16 = 0), bf16 in grad_w by the
register read-add-round epilogue (= 1), and the fp32 accumulator (accum_dtype=torch.float32).
Median over interleaved rounds of ms/step and per-stage ms (lk_profile)."""

import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2410_10989_b200 import _capi  # noqa: E402
from paper_2410_10989_b200.fused_linear_cross_entropy import fused_linear_cross_entropy_forward as f  # noqa: E402

BT, H, V = 8192, 4096, 128256
g = torch.Generator(device="cuda").manual_seed(0)
x = (torch.rand(BT, H, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
w = ((torch.rand(V, H, device="cuda", generator=g) * 2 - 1) / 64.0).to(torch.bfloat16)
t = torch.randint(0, V, (BT,), device="cuda", generator=g)
t[torch.rand(BT, device="cuda", generator=g) < 0.1] = -100
L = _capi.load()
CONFIGS = [("bf16_tma_reduce", 0, None), ("bf16_register", 1, None), ("fp32_acc", 0, torch.float32)]
ROUNDS = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def measure(knob, accum, steps=5):
    L.lk_test_select_path(_capi.PATH_DW_ACCUM16, knob)
    kw = dict(compute_grad_input=True, compute_grad_weight=True, check_targets=False, accum_dtype=accum)
    f(x, w, t, **kw)
    torch.cuda.synchronize()
    L.lk_profile_enable(1)
    L.lk_profile_collect(None, None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        f(x, w, t, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms4 = (C.c_double * 4)()
    L.lk_profile_collect(ms4, None)
    L.lk_profile_enable(0)
    L.lk_test_select_path(_capi.PATH_DW_ACCUM16, 0)
    return [e0.elapsed_time(e1) / steps] + [m / steps for m in ms4]


ref = None
res = {c[0]: [] for c in CONFIGS}
for r in range(ROUNDS):
    for name, knob, accum in CONFIGS:
        res[name].append(measure(knob, accum))
for name, knob, accum in CONFIGS:  # the gradients of each config against the fp32 accumulator's
    L.lk_test_select_path(_capi.PATH_DW_ACCUM16, knob)
    gw = f(x, w, t, compute_grad_input=True, compute_grad_weight=True, accum_dtype=accum)[5].float()
    L.lk_test_select_path(_capi.PATH_DW_ACCUM16, 0)
    if ref is None:
        ref = f(x, w, t, compute_grad_input=True, compute_grad_weight=True, accum_dtype=torch.float32)[5].float()
    rs = res[name]
    med = [sorted(col)[len(col) // 2] for col in zip(*rs)]
    ms, lg, fin, bw, oth = med
    print(json.dumps({"config": name, "ms_step": round(ms, 3), "tok_s": round(BT / ms * 1e3), "logits": round(lg, 3),
                      "finalize": round(fin, 3), "backward": round(bw, 3), "gap": round(ms - lg - fin - bw - oth, 3),
                      "dw_max_abs_diff_vs_fp32_acc": float((gw - ref).abs().max())}), flush=True)
