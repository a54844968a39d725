"""Generate golden vectors by running the reference package `rowfuse` itself.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
It imports /root/reference/pkg/src/rowfuse read-only and writes
tests/golden/rowfuse_golden.npz.  The GPU box never reads /root/reference;
tests compare against the committed .npz.

Cases (inputs are generated from seeds the way the reference tests do,
rng.uniform(-1, 1), W scaled by 1/sqrt(H), tests/test_flce.py:30-35):
  ce_kat_*         hand KATs of tests/test_ops.py:309-320
  ce_rand_*        random rows incl. the multi-segment V = 8229 case (tests/test_ops.py:351-361)
  flce_small_c*    BT=64, H=16, V=50 at chunk rows {1, 8, 64} (SPEC.md flce example)
  flce_mid         BT=128, H=64, V=512, f64, reference plan
  flce_cfg1        cfg1 (BT=1024, H=512, V=4096, seed 0, f64): loss + checksums + sampled entries
  flce_scalar      BT=6, H=5, V=7 through the scalar oracle ref_linear_cross_entropy
  rms_*, ln_*, rope_*, swiglu_*, geglu_*  row ops at f64
  plan_table       chunk-size table of tests/test_flce.py:40-53
  converge_*       loss curves of rowfuse.converge.converge() (100 SGD steps, f32, fused and baseline)
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "rowfuse_golden.npz"


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    from rowfuse import oracle  # noqa: E402
    from rowfuse.core import DType, Matrix2D, Vector  # noqa: E402
    from rowfuse.flce import ChunkPlan, ProjectionHead, flce_forward_backward, plan_chunks  # noqa: E402
    from rowfuse.ops import (  # noqa: E402
        GluInputs,
        Reduction,
        RotationSpec,
        cross_entropy,
        geglu_backward,
        geglu_forward,
        layernorm_backward,
        layernorm_forward,
        rmsnorm_backward,
        rmsnorm_forward,
        rope_backward,
        rope_forward,
        rotation_thetas,
        swiglu_backward,
        swiglu_forward,
    )

    g: dict[str, np.ndarray] = {}

    # ---- cross entropy KATs ----
    def ce(logits, t, red):
        m = Matrix2D.from_array(np.array(logits, dtype=np.float64))
        res = cross_entropy(m, np.array(t), red)
        return res.loss, m.view2d.copy()

    loss, grad = ce([[0.0, 0.0, 0.0, 0.0]], [2], Reduction.SUM)
    g["ce_kat_1_logits"] = np.zeros((1, 4)); g["ce_kat_1_target"] = np.array([2])
    g["ce_kat_1_loss"] = np.array(loss); g["ce_kat_1_grad"] = grad
    loss, grad = ce([[1.0, 2.0]], [1], Reduction.SUM)
    g["ce_kat_2_logits"] = np.array([[1.0, 2.0]]); g["ce_kat_2_target"] = np.array([1])
    g["ce_kat_2_loss"] = np.array(loss); g["ce_kat_2_grad"] = grad

    for name, rows, vocab, seed, red in (("a", 16, 37, 1, Reduction.MEAN), ("b", 4, 8229, 2, Reduction.MEAN),
                                         ("c", 33, 1000, 3, Reduction.SUM)):
        rng = np.random.default_rng(seed)
        x = rng.uniform(-4, 4, (rows, vocab))
        t = rng.integers(0, vocab, rows)
        loss, grad = ce(x, t, red)
        g[f"ce_rand_{name}_logits"] = x; g[f"ce_rand_{name}_target"] = t
        g[f"ce_rand_{name}_mean"] = np.array(red is Reduction.MEAN)
        g[f"ce_rand_{name}_loss"] = np.array(loss); g[f"ce_rand_{name}_grad"] = grad

    # ---- FLCE ----
    def problem(bt, h, v, seed):
        rng = np.random.default_rng(seed)
        x = rng.uniform(-1, 1, (bt, h))
        w = rng.uniform(-1, 1, (h, v)) / math.sqrt(h)
        t = rng.integers(0, v, bt)
        return x, w, t

    def run_flce(x, w, t, chunk=None, red=Reduction.MEAN):
        head = ProjectionHead.from_weight(Matrix2D.from_array(w.copy()))
        plan = ChunkPlan.with_chunk_rows(x.shape[0], chunk) if chunk else None
        loss, dx, dw = flce_forward_backward(Matrix2D.from_array(x.copy()), head, t, red, plan=plan)
        return loss, dx.view2d.copy(), dw.view2d.copy()

    x, w, t = problem(64, 16, 50, 0)
    g["flce_small_x"], g["flce_small_w_hv"], g["flce_small_t"] = x, w, t
    for c in (1, 8, 64):
        loss, dx, dw = run_flce(x, w, t, c)
        g[f"flce_small_c{c}_loss"], g[f"flce_small_c{c}_dx"], g[f"flce_small_c{c}_dw_hv"] = np.array(loss), dx, dw

    x, w, t = problem(128, 64, 512, 5)
    loss, dx, dw = run_flce(x, w, t)
    g["flce_mid_x"], g["flce_mid_w_hv"], g["flce_mid_t"] = x, w, t
    g["flce_mid_loss"], g["flce_mid_dx"], g["flce_mid_dw_hv"] = np.array(loss), dx, dw
    loss, dx, dw = run_flce(x, w, t, red=Reduction.SUM)
    g["flce_mid_sum_loss"], g["flce_mid_sum_dx"] = np.array(loss), dx

    # cfg1: X ~ U(-1,1) (1024, 512), W ~ U(-1,1)/sqrt(512) as (H, V), seed 0
    x, w, t = problem(1024, 512, 4096, 0)
    loss, dx, dw = run_flce(x, w, t)
    rng = np.random.default_rng(123)
    ix = rng.integers(0, dx.size, 64)
    iw = rng.integers(0, dw.size, 64)
    g["flce_cfg1_loss"] = np.array(loss)
    g["flce_cfg1_dx_sum"] = np.array(dx.sum()); g["flce_cfg1_dx_abssum"] = np.array(np.abs(dx).sum())
    g["flce_cfg1_dw_sum"] = np.array(dw.sum()); g["flce_cfg1_dw_abssum"] = np.array(np.abs(dw).sum())
    g["flce_cfg1_dx_idx"], g["flce_cfg1_dx_val"] = ix, dx.reshape(-1)[ix]
    g["flce_cfg1_dw_hv_idx"], g["flce_cfg1_dw_hv_val"] = iw, dw.reshape(-1)[iw]

    x, w, t = problem(6, 5, 7, 9)
    loss, dx, dw = oracle.ref_linear_cross_entropy(x, w, t)
    g["flce_scalar_x"], g["flce_scalar_w_hv"], g["flce_scalar_t"] = x, w, t
    g["flce_scalar_loss"], g["flce_scalar_dx"], g["flce_scalar_dw_hv"] = np.array(loss), dx, dw

    # ---- RMSNorm ----
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, (16, 33))
    gam = np.abs(rng.uniform(-1, 1, 33)) + 0.5
    dy = rng.uniform(-1, 1, (16, 33))
    y, res = rmsnorm_forward(Matrix2D.from_array(x), Vector(gam, DType.F64), eps=1e-6)
    dx, dgam = rmsnorm_backward(Matrix2D.from_array(dy), res, Vector(gam, DType.F64))
    g["rms_x"], g["rms_gamma"], g["rms_dy"] = x, gam, dy
    g["rms_y"], g["rms_rstd"], g["rms_dx"], g["rms_dgamma"] = y.view2d.copy(), res.inv_rms.copy(), dx.view2d.copy(), dgam.data.copy()
    g["rms_kat_y"] = rmsnorm_forward(Matrix2D.from_array(np.array([[3.0, 4.0]])), Vector(np.ones(2), DType.F64), eps=0.0)[0].view2d.copy()

    # ---- LayerNorm ----
    rng = np.random.default_rng(14)
    x = rng.uniform(-1, 1, (16, 40)) + 0.3
    gam = np.abs(rng.uniform(-1, 1, 40)) + 0.5
    bet = rng.uniform(-0.5, 0.5, 40)
    dy = rng.uniform(-1, 1, (16, 40))
    y, res = layernorm_forward(Matrix2D.from_array(x), Vector(gam, DType.F64), Vector(bet, DType.F64), eps=1e-6)
    dx, dgam, dbet = layernorm_backward(Matrix2D.from_array(dy), res, Vector(gam, DType.F64))
    g["ln_x"], g["ln_gamma"], g["ln_beta"], g["ln_dy"] = x, gam, bet, dy
    g["ln_y"], g["ln_mean"], g["ln_rstd"] = y.view2d.copy(), res.mean.copy(), res.inv_rms.copy()
    g["ln_dx"], g["ln_dgamma"], g["ln_dbeta"] = dx.view2d.copy(), dgam.data.copy(), dbet.data.copy()

    # ---- RoPE (per-row positions + thetas) ----
    rng = np.random.default_rng(12)
    d = 8
    q = rng.uniform(-1, 1, (12, d)); k = rng.uniform(-1, 1, (12, d))
    th = rotation_thetas(d)
    pos = rng.integers(0, 50, 12).astype(np.float64)
    spec = RotationSpec(d, th, pos)
    qo, ko = rope_forward(Matrix2D.from_array(q), Matrix2D.from_array(k), spec)
    qb, kb = rope_backward(Matrix2D.from_array(q), Matrix2D.from_array(k), spec)
    g["rope_q"], g["rope_k"], g["rope_thetas"], g["rope_pos"] = q, k, th, pos
    g["rope_q_fwd"], g["rope_k_fwd"], g["rope_q_bwd"], g["rope_k_bwd"] = qo.view2d.copy(), ko.view2d.copy(), qb.view2d.copy(), kb.view2d.copy()

    # ---- GLU ----
    rng = np.random.default_rng(13)
    x1 = rng.uniform(-6, 6, (7, 19)); x2 = rng.uniform(-2, 2, (7, 19)); dy = rng.uniform(-1, 1, (7, 19))
    gi = GluInputs(Matrix2D.from_array(x1), Matrix2D.from_array(x2))
    g["glu_x1"], g["glu_x2"], g["glu_dy"] = x1, x2, dy
    g["swiglu_y"] = swiglu_forward(gi).view2d.copy()
    a, b = swiglu_backward(Matrix2D.from_array(dy), gi)
    g["swiglu_dx1"], g["swiglu_dx2"] = a.view2d.copy(), b.view2d.copy()
    g["geglu_y"] = geglu_forward(gi).view2d.copy()
    a, b = geglu_backward(Matrix2D.from_array(dy), gi)
    g["geglu_dx1"], g["geglu_dx2"] = a.view2d.copy(), b.view2d.copy()

    # ---- training parity harness (rowfuse/converge.py): the reference's own loss curves ----
    from rowfuse.converge import ConvergeConfig, converge  # noqa: E402

    rep = converge(ConvergeConfig())
    assert rep.passed
    g["converge_losses_fused"] = np.array(rep.losses_a, dtype=np.float64)
    g["converge_losses_reference"] = np.array(rep.losses_b, dtype=np.float64)

    # ---- chunk plan table ----
    table = [(4096, 131072, 4096), (4096, 32000, 4096), (4096, 40960, 512), (1, 50000, 768), (100, 768, 768),
             (128, 768, 768), (8192, 256000, 4096), (2048, 128256, 4096), (17, 1000, 64), (1000, 999, 1000),
             (3, 7, 2), (64, 64, 64), (8192, 128256, 4096), (65536, 128256, 4096), (1024, 4096, 512),
             (8192, 256000, 3584)]
    g["plan_table"] = np.array([(bt, v, h, plan_chunks(bt, v, h).chunk_rows) for bt, v, h in table], dtype=np.int64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
