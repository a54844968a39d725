"""Stage times of the cfg2 FLCE with and without ignored-row skipping, over chunk sizes (GPU).

    python scripts/skip_chunk_probe.py
Prints one JSON line per (skip, chunk_rows): the median over interleaved rounds of ms/step
(CUDA events over 5 steps after a warm-up call), the per-stage ms from lk_profile, and the GEMM
TFLOP/s on the executed FLOPs."""

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
kept = int((t != -100).sum().item())
L = _capi.load()
CONFIGS = [(False, 2048), (True, 2048), (True, 2560), (True, 1792)]
ROUNDS = int(sys.argv[1]) if len(sys.argv) > 1 else 6
if len(sys.argv) > 2:  # e.g. "0:2048,0:2304,1:2560" = (skip, chunk_rows) pairs
    CONFIGS = [(bool(int(a)), int(b)) for a, b in (c.split(":") for c in sys.argv[2].split(","))]


def measure(skip, chunk, steps=5):
    kw = dict(compute_grad_input=True, compute_grad_weight=True, check_targets=False, skip_ignored_rows=skip,
              chunk_rows=chunk)
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
    return [e0.elapsed_time(e1) / steps] + [m / steps for m in ms4]


res = {c: [] for c in CONFIGS}
for r in range(ROUNDS):  # interleaved: clock drift under the power cap hits every config alike
    for c in CONFIGS:
        res[c].append(measure(*c))
for (skip, chunk), rs in res.items():
    med = [sorted(col)[len(col) // 2] for col in zip(*rs)]
    ms, lg, fin, bw, oth = med
    rows = kept if skip else BT
    print(json.dumps({"skip": skip, "chunk": chunk, "ms_step": round(ms, 3), "tok_s": round(BT / ms * 1e3),
                      "logits": round(lg, 3), "finalize": round(fin, 3), "backward": round(bw, 3),
                      "other": round(oth, 3), "gap": round(ms - lg - fin - bw - oth, 3),
                      "gemm_tflops_exec": round(6.0 * rows * H * V / ((lg + bw) / 1e3) / 1e12, 1)}), flush=True)
