"""float64 restatement of the Liger semantics rowfuse lacks (TEST INFRASTRUCTURE ONLY).

rowfuse has no ignore_index, label smoothing, softcap, z-loss or reduction='none'
(rowfuse/ops.py:489-499 rejects -100).  These functions extend the
reference math (rowfuse/ops.py:502-560, flce.py:107-173) with the semantics the
north star names, written from Liger's published definitions
(LK = liger_kernel 0.8.0, third-party, not vendored in /root/reference):
  ignored rows: zero loss, zero gradient          LK/ops/cross_entropy.py:100-112
  softcap z -> cap*tanh(z/cap), chain (1 - t^2)   LK/ops/cross_entropy.py:133-134, 240-244
  label smoothing eps = ls/V                      LK/ops/cross_entropy.py:136-175, 263-276
  z-loss lse_square_scale * lse^2                 LK/ops/cross_entropy.py:278-289
  MEAN divides by the non-ignored count           LK/ops/cross_entropy.py:218-219, 282-288
Where no option is active the results coincide with rowfuse (pinned in
tests/test_oracle.py), and the extension is cross-checked against torch-CPU
float64 F.cross_entropy.
"""

from __future__ import annotations

import numpy as np


def ce(logits, target, ignore_index=-100, label_smoothing=0.0, lse_square_scale=0.0, softcap=None,
       reduction="mean", token_scaling=False, weight=None):
    """Returns (loss, loss_rows, z_loss, grad) in float64. loss is a scalar unless reduction='none'.

    token_scaling: Liger FLCE use_token_scaling (LK/ops/fused_linear_cross_entropy.py:109-139,
    187-206): each row's loss, z-loss and gradient times its detached target probability.
    weight: class weights (LK/ops/cross_entropy.py:122-124, 165-171, 220-239, 278-288):
    loss_i = (1-ls) w[y_i](lse - z_y) + eps sum_c w_c (lse - z_c), MEAN over sum_valid w[y_i];
    z-loss still over the count (torch F.cross_entropy(weight=, label_smoothing=) semantics)."""
    z = np.asarray(logits, dtype=np.float64)
    y = np.asarray(target, dtype=np.int64)
    rows, vocab = z.shape
    valid = y != ignore_index
    n = int(valid.sum())
    if softcap is not None:
        t = np.tanh(z / softcap)
        zc = softcap * t
    else:
        t = None
        zc = z
    m = zc.max(axis=1, keepdims=True) if vocab else np.zeros((rows, 1))
    e = np.exp(zc - m)
    s = e.sum(axis=1, keepdims=True)
    lse = (m + np.log(s))[:, 0]
    ysafe = np.where(valid, y, 0)
    zy = zc[np.arange(rows), ysafe]
    eps = label_smoothing / vocab
    loss = lse - zy
    if label_smoothing > 0:
        loss = loss * (1.0 - label_smoothing) + (label_smoothing * lse - eps * zc.sum(axis=1))
    zl = lse_square_scale * lse * lse
    scale = 1.0 / max(n, 1) if reduction == "mean" else 1.0
    ts = np.exp(zy - lse) if token_scaling else np.ones(rows)  # per row, detached
    if weight is not None:
        wv = np.asarray(weight, dtype=np.float64)
        wy = np.where(valid, wv[ysafe], 0.0)
        swn = wy.sum() if reduction == "mean" else 1.0
        s1 = ts / (swn if swn != 0 else 1.0)
        s2 = ts * scale
        ls = label_smoothing
        base = (1.0 - ls) * wy * (lse - zy) + eps * (wv[None, :] * (lse[:, None] - zc)).sum(axis=1)
        loss = base * s1 + zl * s2
        zl = zl * s2
        loss = np.where(valid, loss, 0.0)
        zl = np.where(valid, zl, 0.0)
        p = e / s
        g = p * (((1.0 - ls) * wy + eps * wv.sum()) * s1 + 2.0 * lse_square_scale * lse * s2)[:, None]
        g -= eps * wv[None, :] * s1[:, None] if np.ndim(s1) else eps * wv[None, :] * s1
        g[np.arange(rows), ysafe] -= np.where(valid, (1.0 - ls) * wy * s1, 0.0)
        if t is not None:
            g *= 1.0 - t * t
        g[~valid] = 0.0
        if reduction == "none":
            return loss, loss, zl, g
        return float(loss.sum()), loss, float(zl.sum()), g
    scale = scale * ts
    loss = (loss + zl) * scale
    zl = zl * scale
    loss = np.where(valid, loss, 0.0)
    zl = np.where(valid, zl, 0.0)
    p = e / s
    g = p * (1.0 + 2.0 * lse_square_scale * lse[:, None]) - eps
    g[np.arange(rows), ysafe] -= np.where(valid, 1.0 - label_smoothing, 0.0)
    g *= scale[:, None] if np.ndim(scale) else scale
    if t is not None:
        g *= 1.0 - t * t
    g[~valid] = 0.0
    if reduction == "none":
        return loss, loss, zl, g
    return float(loss.sum()), loss, float(zl.sum()), g


def flce(x, weight_vh, target, bias=None, **kw):
    """Unchunked linear + CE in float64 with the Liger (V, H) layout.

    Returns (loss, loss_rows, z_loss, grad_x, grad_w, grad_bias)."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(weight_vh, dtype=np.float64)
    logits = x @ w.T
    if bias is not None:
        logits = logits + np.asarray(bias, dtype=np.float64)
    loss, rows, zl, g = ce(logits, target, **kw)
    gb = g.sum(axis=0) if bias is not None else None
    return loss, rows, zl, g @ w, g.T @ x, gb


def rmsnorm_fwd(x, w, eps=1e-6, offset=0.0):
    """y = x / rms(x) * (offset + w); returns (y, rstd) (LK/ops/rms_norm.py:45-112, all float64)."""
    x = np.asarray(x, dtype=np.float64)
    r = 1.0 / np.sqrt((x * x).mean(axis=1) + eps)
    y = x * r[:, None]
    if w is not None:
        y = y * (offset + np.asarray(w, dtype=np.float64))
    return y, r


def rmsnorm_bwd(dy, x, w, eps=1e-6, offset=0.0):
    """(dx, dw) of rmsnorm_fwd in float64 (LK/ops/rms_norm.py:115-210)."""
    x = np.asarray(x, dtype=np.float64)
    dy = np.asarray(dy, dtype=np.float64)
    n = x.shape[1]
    r = 1.0 / np.sqrt((x * x).mean(axis=1) + eps)
    wo = (offset + np.asarray(w, dtype=np.float64)) if w is not None else 1.0
    m = dy * wo
    dot = (m * x).sum(axis=1)
    dx = r[:, None] * m - (r ** 3 * dot / n)[:, None] * x
    dw = (dy * x * r[:, None]).sum(axis=0) if w is not None else None
    return dx, dw


def rope(q, k, cos, sin, backward=False):
    """q (B, nq, T, d), k (B, nk, T, d), cos/sin (1 or B, T, d) -> rotated copies (LK/ops/rope.py:90-112)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    d = q.shape[-1]
    c = np.asarray(cos, dtype=np.float64)[:, None, :, : d // 2]
    s = np.asarray(sin, dtype=np.float64)[:, None, :, : d // 2]
    if backward:
        s = -s

    def rot(x):
        x1, x2 = x[..., : d // 2], x[..., d // 2 :]
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)

    return rot(q), rot(k)


def rope_tables(seq: int, head_dim: int, base: float = 10000.0, batch: int = 1):
    """HF-style cos/sin tables: cos(pos*theta) tiled on both halves."""
    th = base ** (-2.0 * np.arange(head_dim // 2, dtype=np.float64) / head_dim)
    ang = np.arange(seq, dtype=np.float64)[:, None] * th[None, :]
    emb = np.concatenate([ang, ang], axis=-1)
    cos = np.broadcast_to(np.cos(emb), (batch, seq, head_dim)).copy()
    sin = np.broadcast_to(np.sin(emb), (batch, seq, head_dim)).copy()
    return cos, sin
