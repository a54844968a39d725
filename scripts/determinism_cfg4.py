"""Bitwise run-to-run repeatability of the bf16 FLCE at cfg4 (Gemma-2-9B head, softcap 30,
smoothing 0.1) and cfg2; prints where gx / gw differ between runs."""
import json
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2410_10989_b200.fused_linear_cross_entropy import fused_linear_cross_entropy_forward as f  # noqa: E402


def batch(bt, h, v, seed, wscale):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.rand(bt, h, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(v, h, device="cuda", generator=g) * 2 - 1) * (wscale / 64.0)).to(torch.bfloat16)
    t = torch.randint(0, v, (bt,), device="cuda", generator=g)
    t[torch.rand(bt, device="cuda", generator=g) < 0.1] = -100
    return x, w, t


def diff(a, b):
    d = (a.float() - b.float()).abs()
    nz = (d > 0).nonzero()
    if nz.numel() == 0:
        return None
    rows = nz[:, 0].unique()
    return {"n": int(nz.shape[0]), "max": d.max().item(), "rows": rows[:16].tolist(), "n_rows": int(rows.numel()),
            "cols_first_row": nz[nz[:, 0] == rows[0]][:, 1][:16].tolist()}


for name, (bt, h, v, wscale, kw) in {"cfg4": (8192, 3584, 256000, 30.0, dict(softcap=30.0, label_smoothing=0.1)),
                                     "cfg2": (8192, 4096, 128256, 1.0, {})}.items():
    x, w, t = batch(bt, h, v, 1, wscale)
    ref = None
    for i in range(4):
        loss, _, _, _, gx, gw, _ = f(x, w, t, compute_grad_input=True, compute_grad_weight=True, **kw)
        cur = (loss.item(), gx.clone(), gw.clone())
        if ref is None:
            ref = cur
            continue
        print(json.dumps({"cfg": name, "run": i, "loss_eq": cur[0] == ref[0], "gx": diff(cur[1], ref[1]),
                          "gw": diff(cur[2], ref[2])}), flush=True)
    del x, w, t, ref, cur, gx, gw
    torch.cuda.empty_cache()
