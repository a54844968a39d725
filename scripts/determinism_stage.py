"""Locate the stage of a rare bitwise run-to-run difference in the bf16 FLCE (cfg4 head, one
2048-row chunk): compares the chunk buffer (dZ after the finalize), the tile partials, loss
rows, gx and gw between repeated calls."""
import json
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2410_10989_b200.fused_linear_cross_entropy as F  # noqa: E402

kept = []
_ws = F.workspace


def keep_ws(nbytes, dev):
    t = _ws(nbytes, dev)
    kept.append(t)
    return t


F.workspace = keep_ws


def al(o):
    return (o + 1023) // 1024 * 1024


def run(bt, h, v, wscale, kw, reps, grad_w=True, grad_x=True):
    g = torch.Generator(device="cuda").manual_seed(1)
    x = (torch.rand(bt, h, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(v, h, device="cuda", generator=g) * 2 - 1) * (wscale / 64.0)).to(torch.bfloat16)
    t = torch.randint(0, v, (bt,), device="cuda", generator=g)
    t[torch.rand(bt, device="cuda", generator=g) < 0.1] = -100
    ldz = (v + 63) // 64 * 64
    nparts = (v + 255) // 256
    off_z = al(al(32) + (2 * 1 + 2 + 16) * 4)
    off_p = al(off_z + bt * ldz * 2)
    ref = None
    for i in range(reps):
        kept.clear()
        loss, _, _, _, gx, gw, _ = F.fused_linear_cross_entropy_forward(
            x, w, t, compute_grad_input=grad_x, compute_grad_weight=grad_w, chunk_rows=bt, reduction="none", **kw)
        torch.cuda.synchronize()
        ws = kept[0]
        z = ws[off_z:off_z + bt * ldz * 2].view(torch.bfloat16).view(bt, ldz)[:, :v].clone()
        parts = ws[off_p:off_p + bt * nparts * 16].view(torch.float32).view(bt, nparts, 4).clone()
        cur = dict(loss=loss.clone(), z=z, parts=parts, gx=gx.clone() if grad_x else None,
                   gw=gw.clone() if grad_w else None)
        if ref is None:
            ref = cur
            continue
        out = {"rep": i, "grad_w": grad_w, "grad_x": grad_x}
        for k in cur:
            if cur[k] is None:
                continue
            d = (cur[k].float() - ref[k].float()).abs()
            d = torch.where(torch.isnan(d), torch.zeros_like(d), d)
            nz = (d > 0).nonzero()
            if nz.numel():
                r0 = nz[0, 0].item()
                cols = nz[nz[:, 0] == r0][:, 1] if cur[k].dim() == 2 else nz[:, 0]
                out[k] = {"n": int(nz.shape[0]), "max": d.max().item(), "first": nz[:3].tolist(),
                          "c0": cols[0].item(), "c1": cols[-1].item()}
                if k == "z":
                    out[k]["vals"] = [(ref[k][r0, c].item(), cur[k][r0, c].item()) for c in cols[:4].tolist()]
        print(json.dumps(out), flush=True)


# no gradients: the finalize only reduces the partials, the chunk buffer keeps the logits
run(2048, 3584, 256000, 30.0, dict(softcap=30.0, label_smoothing=0.1), 24, grad_w=False)


def ce_control(rows, v, reps, **kw):
    """standalone CE (two-pass ring) on logits of the same width: repeatability of the ring"""
    import paper_2410_10989_b200 as lk
    g = torch.Generator(device="cuda").manual_seed(2)
    z0 = (torch.randn(rows, v, device="cuda", generator=g) * 10).to(torch.bfloat16)
    t = torch.randint(0, v, (rows,), device="cuda", generator=g)
    t[torch.rand(rows, device="cuda", generator=g) < 0.1] = -100
    ref = None
    for i in range(reps):
        z = z0.clone().requires_grad_(True)
        loss = lk.LigerCrossEntropyLoss(**kw)(z, t)
        loss.backward()
        cur = z.grad.clone()
        if ref is None:
            ref = cur
            continue
        d = (cur.float() - ref.float()).abs()
        nz = (d > 0).nonzero()
        out = {"ce_rep": i, "kw": str(kw)}
        if nz.numel():
            r0 = nz[0, 0].item()
            cols = nz[nz[:, 0] == r0][:, 1]
            out["diff"] = {"n": int(nz.shape[0]), "row": r0, "c0": cols[0].item(), "c1": cols[-1].item(),
                           "vals": [(ref[r0, c].item(), cur[r0, c].item()) for c in cols[:4].tolist()]}
        print(json.dumps(out), flush=True)


if "--ce" in sys.argv:
    ce_control(2048, 256000, 12, softcap=30.0, label_smoothing=0.1)
    ce_control(2048, 256000, 12)
