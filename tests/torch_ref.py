"""Plain PyTorch fp32 reference of FLCE on the GPU (checker for full-size shapes).

The CPU oracle cannot materialise cfg2-sized logits in float64 in seconds, so at
BASELINE sizes the CUDA path is compared with this cuBLAS-fp32 restatement of the
same math (liger_ref.ce), chunked so logits never exceed chunk x V fp32.
"""

import torch


def ce_grad(z, t, ignore_index=-100, label_smoothing=0.0, lse_square_scale=0.0, softcap=None, scale=1.0):
    """Per-row loss and d(loss)/dz for fp32 logits z (rows x V); rows with t == ignore_index -> 0."""
    valid = t != ignore_index
    if softcap is not None:
        th = torch.tanh(z / softcap)
        zc = softcap * th
    else:
        th, zc = None, z
    lse = torch.logsumexp(zc, dim=1)
    tsafe = torch.where(valid, t, torch.zeros_like(t))
    zy = zc.gather(1, tsafe[:, None])[:, 0]
    v = z.shape[1]
    eps = label_smoothing / v
    loss = lse - zy
    if label_smoothing > 0:
        loss = loss * (1 - label_smoothing) + label_smoothing * lse - eps * zc.sum(dim=1)
    zl = lse_square_scale * lse * lse
    loss = (loss + zl) * scale
    p = torch.softmax(zc, dim=1)
    g = p * (1 + 2 * lse_square_scale * lse[:, None]) - eps
    hit = torch.full_like(lse, -(1 - label_smoothing)).masked_fill(~valid, 0.0)  # in z's dtype
    g.scatter_add_(1, tsafe[:, None], hit[:, None])
    g = g * scale
    if th is not None:
        g = g * (1 - th * th)
    g[~valid] = 0
    loss = torch.where(valid, loss, torch.zeros_like(loss))
    return loss, g


def flce_ref(x, w, t, bias=None, ignore_index=-100, label_smoothing=0.0, lse_square_scale=0.0, softcap=None,
             reduction="mean", chunk=2048, compute_dtype=torch.float32):
    """(loss, loss_rows, grad_x, grad_w, grad_bias) in `compute_dtype` (fp32 on the GPU for the
    full-size checks) from (possibly bf16) inputs.  Pinned to oracle.liger_ref by
    tests/test_oracle.py::test_torch_ref_pinned_to_liger_oracle (float64 on CPU)."""
    xf, wf = x.to(compute_dtype), w.to(compute_dtype)
    bt = x.shape[0]
    n = int((t != ignore_index).sum())
    scale = 1.0 / max(n, 1) if reduction == "mean" else 1.0
    gx = torch.empty_like(xf)
    gw = torch.zeros_like(wf)
    gb = torch.zeros(w.shape[0], device=x.device, dtype=compute_dtype) if bias is not None else None
    rows = torch.empty(bt, device=x.device, dtype=compute_dtype)
    for lo in range(0, bt, chunk):
        hi = min(lo + chunk, bt)
        z = xf[lo:hi] @ wf.t()
        if bias is not None:
            z += bias.to(compute_dtype)
        l, g = ce_grad(z, t[lo:hi], ignore_index, label_smoothing, lse_square_scale, softcap, scale)
        rows[lo:hi] = l
        gx[lo:hi] = g @ wf
        gw += g.t() @ xf[lo:hi]
        if gb is not None:
            gb += g.sum(0)
        del z, g
    loss = rows if reduction == "none" else rows.sum()
    return loss, rows, gx, gw, gb


def rel_err(a, b):
    a = a.float()
    b = b.float()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


def close(a, b, rtol):
    """|a-b| <= rtol*(|b| + max|b|) elementwise."""
    a = a.float()
    b = b.float()
    return bool(((a - b).abs() <= rtol * (b.abs() + b.abs().max())).all())
