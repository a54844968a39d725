"""Kept-row FLCE at cfg2: the count read on the host, read ahead (prepare_kept_rows on a side
stream), or kept on the device (KEPT_ROWS_DEVICE_COUNT), interleaved (GPU).

    python scripts/kept_count_probe.py [rounds]"""

import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2410_10989_b200 as lk  # noqa: E402
import paper_2410_10989_b200.fused_linear_cross_entropy as m  # noqa: E402
from paper_2410_10989_b200 import _capi  # noqa: E402

BT, H, V = 8192, 4096, 128256
g = torch.Generator(device="cuda").manual_seed(0)
x = (torch.rand(BT, H, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
w = ((torch.rand(V, H, device="cuda", generator=g) * 2 - 1) / 64.0).to(torch.bfloat16)
t = torch.randint(0, V, (BT,), device="cuda", generator=g)
t[torch.rand(BT, device="cuda", generator=g) < 0.1] = -100
L = _capi.load()
side = torch.cuda.Stream()
ROUNDS = int(sys.argv[1]) if len(sys.argv) > 1 else 8
kw = dict(compute_grad_input=True, compute_grad_weight=True, check_targets=False)


def measure(mode, steps=5):
    m.KEPT_ROWS_DEVICE_COUNT = mode == "device"
    m._PREPARED.clear()
    m.fused_linear_cross_entropy_forward(x, w, t, **kw)
    torch.cuda.synchronize()
    L.lk_profile_enable(1)
    L.lk_profile_collect(None, None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if mode == "prepared":
        lk.prepare_kept_rows(t, stream=side)
    e0.record()
    for _ in range(steps):
        m.fused_linear_cross_entropy_forward(x, w, t, **kw)
        if mode == "prepared":
            lk.prepare_kept_rows(t, stream=side)
    e1.record()
    torch.cuda.synchronize()
    ms4 = (C.c_double * 4)()
    L.lk_profile_collect(ms4, None)
    L.lk_profile_enable(0)
    m.KEPT_ROWS_DEVICE_COUNT = False
    return [e0.elapsed_time(e1) / steps] + [v / steps for v in ms4]


res = {k: [] for k in ("host", "prepared", "device")}
for _ in range(ROUNDS):
    for k in res:
        res[k].append(measure(k))
for k, rs in res.items():
    med = [sorted(c)[len(c) // 2] for c in zip(*rs)]
    ms, lg, fin, bw, oth = med
    print(json.dumps({"count": k, "ms_step": round(ms, 3), "tok_s": round(BT / ms * 1e3), "logits": round(lg, 3),
                      "finalize": round(fin, 3), "backward": round(bw, 3), "other": round(oth, 3),
                      "gap": round(ms - lg - fin - bw - oth, 3)}), flush=True)
