"""numpy restatement of the reference `rowfuse` kernels (TEST INFRASTRUCTURE ONLY).

Every function follows one reference function; citations are to
/root/reference/pkg/src/rowfuse/<file>:<line>.  Layouts are rowfuse's: the head
weight is (H, V) (flce.py:81-104) and RoPE takes per-row positions plus a theta
vector (ops.py:61-89).  The arithmetic runs in the dtype of the inputs, so the
same code is the f64 oracle and (at f32) the timed CPU baseline "port".
"""

from __future__ import annotations

import math

import numpy as np

CE_SEGMENT = 8192          # rowfuse/ops.py:35
GELU_C = math.sqrt(2.0 / math.pi)   # rowfuse/ops.py:37
GELU_A = 0.044715                   # rowfuse/ops.py:38
GELU_3A = 0.134145                  # rowfuse/ops.py:39


class TargetOutOfRange(IndexError):
    """rowfuse/core.py:45-46."""


# --------------------------------------------------------------- planning --
def next_pow2(n: int) -> int:
    """rowfuse/flce.py:31-32."""
    return 1 if n <= 1 else 1 << (n - 1).bit_length()


def plan_chunk_rows(total_rows: int, vocab: int, hidden: int) -> int:
    """rowfuse/flce.py:69-78: 2^ceil(log2(ceil(BT / ceil(V/H))))."""
    per = -(-vocab // hidden)
    return next_pow2(-(-total_rows // per))


# ----------------------------------------------------------- cross entropy --
def check_targets(targets, rows: int, vocab: int) -> np.ndarray:
    """rowfuse/ops.py:489-499."""
    t = np.asarray(targets)
    if t.ndim != 1 or t.shape[0] != rows:
        raise ValueError(f"need one target per row ({rows}), got shape {t.shape}")
    t = t.astype(np.int64)
    if t.size and (t.min() < 0 or t.max() >= vocab):
        raise TargetOutOfRange(f"target outside [0, {vocab})")
    return t


def cross_entropy_(logits: np.ndarray, targets, mean: bool = True) -> float:
    """In-place streaming softmax cross entropy (rowfuse/ops.py:502-560).

    For every row: running (max, sum-exp) over CE_SEGMENT-wide segments with
    rescaling when the max grows (533-545), then the row is rewritten to
    exp(x - m) / s and the target entry lowered by one (547-551).  The loss uses
    a clamped log (550).  MEAN divides loss and buffer by the row count (557-559).
    Returns the loss; `logits` holds d(loss)/d(logits) afterwards.
    """
    rows, vocab = logits.shape
    t = check_targets(targets, rows, vocab)
    tiny = float(np.finfo(logits.dtype).tiny)
    seg = min(vocab, CE_SEGMENT)
    work = np.empty(seg, dtype=logits.dtype)
    losses = np.empty(rows, dtype=np.float64)
    for i in range(rows):
        row = logits[i]
        m, s = -math.inf, 0.0
        for lo in range(0, vocab, seg):
            hi = min(lo + seg, vocab)
            blk_max = float(row[lo:hi].max())
            if blk_max > m:
                s = s * math.exp(m - blk_max) if s > 0.0 else s
                m = blk_max
            w = work[: hi - lo]
            np.subtract(row[lo:hi], m, out=w)
            np.exp(w, out=w)
            s += float(w.sum())
        np.subtract(row, m, out=row)
        np.exp(row, out=row)
        np.divide(row, s, out=row)
        losses[i] = -math.log(max(float(row[t[i]]), tiny))
        row[t[i]] -= 1.0
    total = math.fsum(losses)
    if mean:
        total /= rows
        np.divide(logits, rows, out=logits)
    return float(total)


# -------------------------------------------------------------------- FLCE --
def flce_forward_backward(hidden: np.ndarray, weight_hv: np.ndarray, targets, mean: bool = True,
                          chunk_rows: int | None = None):
    """Chunked projection head (rowfuse/flce.py:107-173).

    hidden (BT, H), weight_hv (H, V) -> (loss, dhidden (BT, H), dweight (H, V)).
    One (chunk x V) scratch is reused: logits GEMM (153), in-place CE with SUM
    (155-157), dX GEMM (160), dW accumulate (161-162); MEAN is applied once after
    the loop (165-168) so the result is independent of the chunk schedule.
    """
    bt, h = hidden.shape
    h2, vocab = weight_hv.shape
    if h2 != h:
        raise ValueError(f"hidden width {h} != head input width {h2}")
    t = check_targets(targets, bt, vocab)
    c = chunk_rows or plan_chunk_rows(bt, vocab, h)
    dt = hidden.dtype
    dw = np.zeros((h, vocab), dtype=dt)
    dx = np.empty_like(hidden)
    scratch = np.empty((c, vocab), dtype=dt)
    tmp = np.empty((h, vocab), dtype=dt)
    losses = []
    for lo in range(0, bt, c):
        hi = min(lo + c, bt)
        blk = scratch[: hi - lo]
        np.matmul(hidden[lo:hi], weight_hv, out=blk)
        losses.append(cross_entropy_(blk, t[lo:hi], mean=False))
        np.matmul(blk, weight_hv.T, out=dx[lo:hi])
        np.matmul(hidden[lo:hi].T, blk, out=tmp)
        dw += tmp
    total = 0.0
    for v in losses:            # rowfuse/flce.py:176-180 sequential sum
        total += v
    if mean:
        total /= bt
        dx /= bt
        dw /= bt
    return float(total), dx, dw


# ----------------------------------------------------------------- RMSNorm --
def rmsnorm_forward(x: np.ndarray, gamma: np.ndarray, eps: float = 1e-6):
    """rowfuse/ops.py:190-214: y = x * r * gamma, r = 1/sqrt(mean(x^2) + eps); caches r."""
    n = x.shape[1]
    ss = np.einsum("ij,ij->i", x, x)
    r = 1.0 / np.sqrt(ss / n + eps)
    return (x * r[:, None]) * gamma, r.astype(x.dtype)


def tree_sum(parts: np.ndarray) -> np.ndarray:
    """Fixed-order pairwise reduction over axis 0 (rowfuse/ops.py:138-152)."""
    a = parts
    while a.shape[0] > 1:
        n = a.shape[0]
        head = a[0 : n - (n % 2) : 2] + a[1 : n - (n % 2) : 2]
        a = np.concatenate([head, a[n - 1 : n]]) if n % 2 else head
    return a[0].copy()


def rmsnorm_backward(dy: np.ndarray, x: np.ndarray, r: np.ndarray, gamma: np.ndarray):
    """rowfuse/ops.py:217-241: dx = r*(dy*g - (xhat.(dy*g)/n) xhat), dgamma = tree_sum(dy*xhat)."""
    n = x.shape[1]
    xhat = x * r[:, None]
    gy = dy * gamma
    proj = np.einsum("ij,ij->i", xhat, gy) / n
    dx = (gy - proj[:, None] * xhat) * r[:, None]
    return dx, tree_sum(dy * xhat)


# --------------------------------------------------------------- LayerNorm --
def layernorm_forward(x: np.ndarray, gamma: np.ndarray, beta: np.ndarray, eps: float = 1e-6):
    """rowfuse/ops.py:248-275: centred, r = 1/sqrt(mean((x-mu)^2) + eps); caches (mu, r)."""
    n = x.shape[1]
    mu = x.mean(axis=1)
    v = x - mu[:, None]
    r = 1.0 / np.sqrt(np.einsum("ij,ij->i", v, v) / n + eps)
    return v * r[:, None] * gamma + beta, mu.astype(x.dtype), r.astype(x.dtype)


def layernorm_backward(dy: np.ndarray, x: np.ndarray, mu: np.ndarray, r: np.ndarray, gamma: np.ndarray):
    """rowfuse/ops.py:278-311: dx = r (gy - (xt.gy/n) xt - sum(gy)/n); dgamma, dbeta tree sums."""
    n = x.shape[1]
    xt = (x - mu[:, None]) * r[:, None]
    gy = dy * gamma
    proj = np.einsum("ij,ij->i", xt, gy) / n
    shift = gy.sum(axis=1) / n
    dx = (gy - proj[:, None] * xt - shift[:, None]) * r[:, None]
    return dx, tree_sum(dy * xt), tree_sum(dy)


# -------------------------------------------------------------------- RoPE --
def rotation_thetas(head_dim: int, base: float = 10000.0) -> np.ndarray:
    """rowfuse/ops.py:85-89: base^(-2i/d)."""
    return base ** (-2.0 * np.arange(head_dim // 2, dtype=np.float64) / head_dim)


def rope_apply(x: np.ndarray, thetas: np.ndarray, positions: np.ndarray, backward: bool = False) -> np.ndarray:
    """Half-split rotation by pos*theta per row (rowfuse/ops.py:322-382); backward negates sin."""
    dt = x.dtype
    ang = positions.astype(dt)[:, None] * thetas.astype(dt)[None, :]
    cos, sin = np.cos(ang), np.sin(ang)
    if backward:
        sin = -sin
    half = thetas.shape[0]
    x1, x2 = x[:, :half], x[:, half:]
    out = np.empty_like(x)
    out[:, :half] = x1 * cos - x2 * sin
    out[:, half:] = x1 * sin + x2 * cos
    return out


# --------------------------------------------------------------------- GLU --
def sigmoid(z: np.ndarray) -> np.ndarray:
    """Overflow-safe logistic (rowfuse/ops.py:155-162)."""
    e = np.exp(-np.abs(z))
    return np.where(z >= 0, 1.0, e) / (1.0 + e)


def swiglu_forward(x1, x2):
    """rowfuse/ops.py:389-402."""
    return x1 * sigmoid(x1) * x2


def swiglu_backward(dy, x1, x2):
    """rowfuse/ops.py:405-430: dx1 = dy*(sig + silu*(1-sig))*x2, dx2 = dy*silu."""
    sg = sigmoid(x1)
    silu = x1 * sg
    return dy * (sg + silu * (1.0 - sg)) * x2, dy * silu


def gelu_tanh(z):
    """rowfuse/ops.py:433-435."""
    t = np.tanh(GELU_C * (z + GELU_A * z ** 3))
    return 0.5 * z * (1.0 + t), t


def geglu_forward(x1, x2):
    """rowfuse/ops.py:438-451."""
    return gelu_tanh(x1)[0] * x2


def geglu_backward(dy, x1, x2):
    """rowfuse/ops.py:454-482."""
    g, t = gelu_tanh(x1)
    dg = 0.5 * (1.0 + t) + 0.5 * GELU_C * x1 * (1.0 - t * t) * (1.0 + GELU_3A * x1 * x1)
    return dy * dg * x2, dy * g
