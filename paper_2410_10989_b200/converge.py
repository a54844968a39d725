"""Training-parity harness on the GPU (rowfuse/converge.py:1-315).

The reference's end-to-end gate: a tiny decoder -- token embedding, two pre-norm blocks
(RMSNorm -> SwiGLU / GeGLU MLP -> rotation-only attention stub), a final LayerNorm and
the chunked linear cross-entropy head -- trained with plain SGD on a fixed synthetic
token stream, two ways from identical initial parameters:

  path "fused"     : every kernel of this library (RMSNorm, SwiGLU, GeGLU, RoPE,
                     LayerNorm, FLCE) through its Liger autograd Function on cuda:0;
  path "reference" : plain torch autograd in the same dtype (unfused, full logits).

Loss curves, final parameters and final logits must agree within (atol, rtol)
(rowfuse/converge.py:283-315).  Parameters, data and the model are the reference's
exactly (same seeds and draw order, rowfuse/converge.py:80-108), so the fused loss curve
can also be compared with the reference's own numpy run (tests/golden converge_* arrays).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F


@dataclass
class ConvergeConfig:  # rowfuse/converge.py:53-66
    steps: int = 100
    seed: int = 0
    dtype: torch.dtype = torch.float32
    lr: float = 0.1
    vocab: int = 64
    hidden: int = 16
    mlp: int = 32
    batch: int = 4
    seqlen: int = 16
    atol: float = 1e-5
    rtol: float = 1e-4
    device: str = "cuda"


@dataclass
class ConvergenceReport:  # rowfuse/converge.py:69-77
    steps: int
    losses_a: list = field(default_factory=list)
    losses_b: list = field(default_factory=list)
    max_loss_diff: float = 0.0
    final_param_diff: float = 0.0
    final_logits_diff: float = 0.0
    passed: bool = False


def init_params(cfg: ConvergeConfig) -> dict:
    """rowfuse/converge.py:80-101 (same generator, same draw order)."""
    rng = np.random.default_rng(cfg.seed)
    h, m, v = cfg.hidden, cfg.mlp, cfg.vocab

    def mat(r, c, scale):
        return (rng.standard_normal((r, c)) * scale).astype(np.float32)

    p = {"embed": mat(v, h, 0.5), "ln_g": np.ones(h, np.float32), "ln_b": np.zeros(h, np.float32),
         "head": mat(h, v, 1.0 / math.sqrt(h))}
    for b in range(2):
        p[f"g{b}"] = np.ones(h, np.float32)
        p[f"wg{b}"] = mat(h, m, 1.0 / math.sqrt(h))
        p[f"bg{b}"] = np.zeros(m, np.float32)
        p[f"wv{b}"] = mat(h, m, 1.0 / math.sqrt(h))
        p[f"bv{b}"] = np.zeros(m, np.float32)
        p[f"down{b}"] = mat(m, h, 1.0 / math.sqrt(m))
    return p


def make_data(cfg: ConvergeConfig):
    """rowfuse/converge.py:104-110: fixed stream, targets are the next token."""
    rng = np.random.default_rng(cfg.seed + 1)
    tok = rng.integers(0, cfg.vocab, size=(cfg.batch, cfg.seqlen))
    targets = np.roll(tok, -1, axis=1).reshape(-1)
    positions = np.tile(np.arange(cfg.seqlen), cfg.batch)
    return tok.reshape(-1), positions, targets


def rope_tables(cfg: ConvergeConfig, device):
    """cos/sin (1, T, d) of rowfuse's RotationSpec(hidden, thetas(base 1e4), positions)."""
    d = cfg.hidden
    th = 10000.0 ** (-np.arange(0, d, 2, dtype=np.float64) / d)
    ang = np.arange(cfg.seqlen, dtype=np.float64)[:, None] * th[None, :]
    emb = np.concatenate([ang, ang], axis=-1)[None]
    return (torch.tensor(np.cos(emb), dtype=cfg.dtype, device=device),
            torch.tensor(np.sin(emb), dtype=cfg.dtype, device=device))


def _fused_loss(P, tok, tgt, cos, sin, cfg):
    from . import (LigerFusedLinearCrossEntropyFunction, LigerGELUMulFunction, LigerLayerNormFunction,
                   LigerRMSNormFunction, LigerSiLUMulFunction, liger_rotary_pos_emb)

    B, T, H = cfg.batch, cfg.seqlen, cfg.hidden
    x = P["embed"][tok]
    for b in range(2):
        y = LigerRMSNormFunction.apply(x, P[f"g{b}"], 1e-6, 0.0, "llama", False)
        a1 = y @ P[f"wg{b}"] + P[f"bg{b}"]
        a2 = y @ P[f"wv{b}"] + P[f"bv{b}"]
        g = LigerSiLUMulFunction.apply(a1, a2) if b == 0 else LigerGELUMulFunction.apply(a1, a2)
        mid = g @ P[f"down{b}"]
        q = mid.view(B, T, 1, H).transpose(1, 2).clone()
        k = mid.view(B, T, 1, H).transpose(1, 2).clone()
        qr, kr = liger_rotary_pos_emb(q, k, cos, sin)
        x = (0.5 * (qr + kr)).transpose(1, 2).reshape(B * T, H)
    yn = LigerLayerNormFunction.apply(x, P["ln_g"], P["ln_b"], 1e-6)
    loss, _, _, _ = LigerFusedLinearCrossEntropyFunction.apply(
        yn, P["head"].t().contiguous(), tgt, None, None, -100, 0.0, 0.0, "mean", None, False, None, False, False,
        False)
    return loss


def _rot(x, cos, sin):
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    return x * cos + torch.cat([-x2, x1], dim=-1) * sin


def _reference_forward(P, tok, cos, sin, cfg):
    B, T, H = cfg.batch, cfg.seqlen, cfg.hidden
    x = P["embed"][tok]
    for b in range(2):
        y = x * torch.rsqrt((x * x).mean(1, keepdim=True) + 1e-6) * P[f"g{b}"]
        a1 = y @ P[f"wg{b}"] + P[f"bg{b}"]
        a2 = y @ P[f"wv{b}"] + P[f"bv{b}"]
        g = F.silu(a1) * a2 if b == 0 else F.gelu(a1, approximate="tanh") * a2
        mid = (g @ P[f"down{b}"]).view(B, T, H)
        x = _rot(mid, cos, sin).reshape(B * T, H)
    yn = F.layer_norm(x, (H,), P["ln_g"], P["ln_b"], eps=1e-6)
    return yn @ P["head"]


def _reference_loss(P, tok, tgt, cos, sin, cfg):
    return F.cross_entropy(_reference_forward(P, tok, cos, sin, cfg), tgt)


def converge(cfg: ConvergeConfig | None = None) -> ConvergenceReport:
    """Train both copies and report whether their trajectories agree (rowfuse/converge.py:274-315)."""
    cfg = cfg or ConvergeConfig()
    dev = torch.device(cfg.device)
    base = init_params(cfg)
    pa = {k: torch.tensor(v, dtype=cfg.dtype, device=dev, requires_grad=True) for k, v in base.items()}
    pb = {k: torch.tensor(v, dtype=cfg.dtype, device=dev, requires_grad=True) for k, v in base.items()}
    tok, _, tgt = make_data(cfg)
    tok = torch.tensor(tok, device=dev)
    tgt = torch.tensor(tgt, device=dev)
    cos, sin = rope_tables(cfg, dev)
    rep = ConvergenceReport(steps=cfg.steps)
    for _ in range(cfg.steps):
        la = _fused_loss(pa, tok, tgt, cos, sin, cfg)
        lb = _reference_loss(pb, tok, tgt, cos, sin, cfg)
        la.backward()
        lb.backward()
        fa, fb = float(la.item()), float(lb.item())
        if not (math.isfinite(fa) and math.isfinite(fb)):
            raise ArithmeticError(f"non-finite loss: {fa}, {fb}")
        rep.losses_a.append(fa)
        rep.losses_b.append(fb)
        with torch.no_grad():
            for p in list(pa.values()) + list(pb.values()):
                p -= cfg.lr * p.grad
                p.grad = None
    rep.max_loss_diff = max(abs(a - b) for a, b in zip(rep.losses_a, rep.losses_b))
    losses_ok = all(abs(a - b) <= cfg.atol + cfg.rtol * abs(b) for a, b in zip(rep.losses_a, rep.losses_b))
    params_ok, gap_max = True, 0.0
    for k in base:
        a64, b64 = pa[k].detach().double(), pb[k].detach().double()
        gap = (a64 - b64).abs()
        gap_max = max(gap_max, float(gap.max()))
        params_ok = params_ok and bool(torch.all(gap <= cfg.atol + cfg.rtol * b64.abs()))
    rep.final_param_diff = gap_max
    with torch.no_grad():
        za = _reference_forward(pa, tok, cos, sin, cfg).double()
        zb = _reference_forward(pb, tok, cos, sin, cfg).double()
    rep.final_logits_diff = float((za - zb).abs().max())
    logits_ok = bool(torch.all((za - zb).abs() <= cfg.atol + cfg.rtol * zb.abs()))
    rep.passed = losses_ok and params_ok and logits_ok
    return rep
