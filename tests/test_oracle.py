"""Pin the CPU oracle before trusting it (CPU only).

* oracle.rowfuse_port against golden vectors produced by the reference itself
  (tests/golden/make_golden.py imports /root/reference/pkg/src/rowfuse);
* oracle.liger_ref where no Liger option is active against the same goldens, and
  with options (ignore_index, label smoothing, softcap, z-loss, reductions)
  against torch-CPU float64 F.cross_entropy + autograd.
"""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import liger_ref, rowfuse_port as rp
from paper_2410_10989_b200.chunking import ChunkPlan, b200_plan, plan_chunks

STRICT = dict(rtol=1e-10, atol=1e-12)


def test_ce_known_answers(golden):
    for k in (1, 2):
        x = golden[f"ce_kat_{k}_logits"].copy()
        loss = rp.cross_entropy_(x, golden[f"ce_kat_{k}_target"], mean=False)
        assert loss == pytest.approx(float(golden[f"ce_kat_{k}_loss"]), rel=1e-14)
        np.testing.assert_allclose(x, golden[f"ce_kat_{k}_grad"], **STRICT)
    assert float(golden["ce_kat_1_loss"]) == pytest.approx(math.log(4))
    np.testing.assert_allclose(golden["ce_kat_1_grad"], [[0.25, 0.25, -0.75, 0.25]])
    assert float(golden["ce_kat_2_loss"]) == pytest.approx(0.3132617, abs=1e-7)


@pytest.mark.parametrize("case", ["a", "b", "c"])
def test_ce_random_vs_reference(golden, case):
    x = golden[f"ce_rand_{case}_logits"].copy()
    mean = bool(golden[f"ce_rand_{case}_mean"])
    loss = rp.cross_entropy_(x, golden[f"ce_rand_{case}_target"], mean=mean)
    assert loss == pytest.approx(float(golden[f"ce_rand_{case}_loss"]), rel=1e-12)
    np.testing.assert_allclose(x, golden[f"ce_rand_{case}_grad"], **STRICT)
    # rows of the gradient sum to zero (SPEC.md invariant)
    np.testing.assert_allclose(x.sum(axis=1), 0.0, atol=1e-12)


@pytest.mark.parametrize("chunk", [1, 8, 64])
def test_flce_small_vs_reference(golden, chunk):
    loss, dx, dw = rp.flce_forward_backward(golden["flce_small_x"], golden["flce_small_w_hv"],
                                            golden["flce_small_t"], mean=True, chunk_rows=chunk)
    assert loss == pytest.approx(float(golden[f"flce_small_c{chunk}_loss"]), rel=1e-12)
    np.testing.assert_allclose(dx, golden[f"flce_small_c{chunk}_dx"], **STRICT)
    np.testing.assert_allclose(dw, golden[f"flce_small_c{chunk}_dw_hv"], **STRICT)


def test_flce_mid_and_scalar_vs_reference(golden):
    loss, dx, dw = rp.flce_forward_backward(golden["flce_mid_x"], golden["flce_mid_w_hv"], golden["flce_mid_t"])
    assert loss == pytest.approx(float(golden["flce_mid_loss"]), rel=1e-12)
    np.testing.assert_allclose(dx, golden["flce_mid_dx"], **STRICT)
    np.testing.assert_allclose(dw, golden["flce_mid_dw_hv"], **STRICT)
    loss_s, dx_s, _ = rp.flce_forward_backward(golden["flce_mid_x"], golden["flce_mid_w_hv"], golden["flce_mid_t"],
                                               mean=False)
    assert loss_s == pytest.approx(float(golden["flce_mid_sum_loss"]), rel=1e-12)
    np.testing.assert_allclose(dx_s, golden["flce_mid_sum_dx"], **STRICT)
    loss, dx, dw = rp.flce_forward_backward(golden["flce_scalar_x"], golden["flce_scalar_w_hv"],
                                            golden["flce_scalar_t"])
    assert loss == pytest.approx(float(golden["flce_scalar_loss"]), rel=1e-12)
    np.testing.assert_allclose(dx, golden["flce_scalar_dx"], **STRICT)
    np.testing.assert_allclose(dw, golden["flce_scalar_dw_hv"], **STRICT)


def cfg1_problem(seed=0, bt=1024, h=512, v=4096):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (bt, h))
    w = rng.uniform(-1, 1, (h, v)) / math.sqrt(h)
    t = rng.integers(0, v, bt)
    return x, w, t


def test_flce_cfg1_checksums(golden):
    x, w, t = cfg1_problem()
    loss, dx, dw = rp.flce_forward_backward(x, w, t)
    assert loss == pytest.approx(float(golden["flce_cfg1_loss"]), rel=1e-12)
    assert dx.sum() == pytest.approx(float(golden["flce_cfg1_dx_sum"]), rel=1e-9, abs=1e-12)
    assert np.abs(dw).sum() == pytest.approx(float(golden["flce_cfg1_dw_abssum"]), rel=1e-12)
    np.testing.assert_allclose(dx.reshape(-1)[golden["flce_cfg1_dx_idx"]], golden["flce_cfg1_dx_val"], **STRICT)
    np.testing.assert_allclose(dw.reshape(-1)[golden["flce_cfg1_dw_hv_idx"]], golden["flce_cfg1_dw_hv_val"], **STRICT)


def test_liger_ref_matches_reference_without_options(golden):
    x, w_hv, t = golden["flce_mid_x"], golden["flce_mid_w_hv"], golden["flce_mid_t"]
    loss, _, _, gx, gw, _ = liger_ref.flce(x, w_hv.T, t)
    assert loss == pytest.approx(float(golden["flce_mid_loss"]), rel=1e-12)
    np.testing.assert_allclose(gx, golden["flce_mid_dx"], **STRICT)
    np.testing.assert_allclose(gw.T, golden["flce_mid_dw_hv"], **STRICT)


@pytest.mark.parametrize("reduction", ["mean", "sum", "none"])
@pytest.mark.parametrize("ls,cap", [(0.0, None), (0.1, None), (0.0, 30.0), (0.1, 4.0)])
def test_liger_ref_vs_torch_f64(reduction, ls, cap):
    rng = np.random.default_rng(7)
    rows, v = 40, 97
    z = rng.normal(0, 5, (rows, v))
    t = rng.integers(0, v, rows)
    t[rng.random(rows) < 0.2] = -100
    loss, loss_rows, _, g = liger_ref.ce(z, t, ignore_index=-100, label_smoothing=ls, softcap=cap,
                                         reduction=reduction)
    zt = torch.tensor(z, dtype=torch.float64, requires_grad=True)
    zc = cap * torch.tanh(zt / cap) if cap else zt
    tl = F.cross_entropy(zc, torch.tensor(t), ignore_index=-100, label_smoothing=ls, reduction=reduction)
    if reduction == "none":
        np.testing.assert_allclose(loss, tl.detach().numpy(), rtol=1e-12, atol=1e-12)
        tl.sum().backward()
    else:
        assert loss == pytest.approx(tl.item(), rel=1e-12)
        tl.backward()
    np.testing.assert_allclose(g, zt.grad.numpy(), rtol=1e-10, atol=1e-14)


def test_liger_ref_z_loss_gradient():
    rng = np.random.default_rng(3)
    z = rng.normal(0, 2, (9, 13))
    t = rng.integers(0, 13, 9)
    t[0] = -100
    lss = 1e-2
    loss, _, zl, g = liger_ref.ce(z, t, lse_square_scale=lss, reduction="mean")
    zt = torch.tensor(z, requires_grad=True)
    valid = torch.tensor(t != -100)
    lse = torch.logsumexp(zt, dim=1)
    ce = F.cross_entropy(zt, torch.tensor(t), ignore_index=-100, reduction="sum")
    ref = (ce + (lss * lse * lse * valid).sum()) / valid.sum()
    ref.backward()
    assert loss == pytest.approx(ref.item(), rel=1e-12)
    np.testing.assert_allclose(g, zt.grad.numpy(), rtol=1e-10, atol=1e-14)


def test_layernorm_port_vs_reference(golden):
    y, mu, r = rp.layernorm_forward(golden["ln_x"], golden["ln_gamma"], golden["ln_beta"])
    np.testing.assert_allclose(y, golden["ln_y"], **STRICT)
    np.testing.assert_allclose(mu, golden["ln_mean"], **STRICT)
    np.testing.assert_allclose(r, golden["ln_rstd"], **STRICT)
    dx, dg, db = rp.layernorm_backward(golden["ln_dy"], golden["ln_x"], mu, r, golden["ln_gamma"])
    np.testing.assert_allclose(dx, golden["ln_dx"], **STRICT)
    np.testing.assert_array_equal(dg, golden["ln_dgamma"])  # same fixed-order tree: bitwise
    np.testing.assert_array_equal(db, golden["ln_dbeta"])
    # the centred form equals torch's layer_norm (biased variance, eps inside the root)
    import torch

    t = torch.nn.functional.layer_norm(torch.tensor(golden["ln_x"]), (golden["ln_x"].shape[1],),
                                       torch.tensor(golden["ln_gamma"]), torch.tensor(golden["ln_beta"]), eps=1e-6)
    np.testing.assert_allclose(t.numpy(), golden["ln_y"], **STRICT)


def test_rmsnorm_port_vs_reference(golden):
    y, r = rp.rmsnorm_forward(golden["rms_x"], golden["rms_gamma"])
    np.testing.assert_allclose(y, golden["rms_y"], **STRICT)
    np.testing.assert_allclose(r, golden["rms_rstd"], **STRICT)
    dx, dg = rp.rmsnorm_backward(golden["rms_dy"], golden["rms_x"], r, golden["rms_gamma"])
    np.testing.assert_allclose(dx, golden["rms_dx"], **STRICT)
    np.testing.assert_array_equal(dg, golden["rms_dgamma"])  # same fixed-order tree: bitwise
    y2, _ = liger_ref.rmsnorm_fwd(golden["rms_x"], golden["rms_gamma"])
    np.testing.assert_allclose(y2, golden["rms_y"], **STRICT)
    dx2, dg2 = liger_ref.rmsnorm_bwd(golden["rms_dy"], golden["rms_x"], golden["rms_gamma"])
    np.testing.assert_allclose(dx2, golden["rms_dx"], **STRICT)
    np.testing.assert_allclose(dg2, golden["rms_dgamma"], **STRICT)
    np.testing.assert_allclose(golden["rms_kat_y"], [[0.8485281, 1.1313708]], atol=1e-7)


def test_rope_port_vs_reference(golden):
    q, k, th, pos = golden["rope_q"], golden["rope_k"], golden["rope_thetas"], golden["rope_pos"]
    np.testing.assert_allclose(rp.rope_apply(q, th, pos), golden["rope_q_fwd"], **STRICT)
    np.testing.assert_allclose(rp.rope_apply(k, th, pos), golden["rope_k_fwd"], **STRICT)
    np.testing.assert_allclose(rp.rope_apply(q, th, pos, backward=True), golden["rope_q_bwd"], **STRICT)
    # norm preservation and inverse (SPEC.md invariants)
    y = rp.rope_apply(q, th, pos)
    np.testing.assert_allclose(np.linalg.norm(y, axis=1), np.linalg.norm(q, axis=1), rtol=1e-12)
    np.testing.assert_allclose(rp.rope_apply(y, th, pos, backward=True), q, atol=1e-12)


def test_rope_tables_adapter_matches_port():
    # cos/sin tables (Liger) == per-row positions + thetas (rowfuse), SURVEY Appendix B.7
    rng = np.random.default_rng(4)
    b, nq, nk, tlen, d = 2, 4, 2, 6, 8
    q = rng.uniform(-1, 1, (b, nq, tlen, d))
    k = rng.uniform(-1, 1, (b, nk, tlen, d))
    cos, sin = liger_ref.rope_tables(tlen, d)
    qo, ko = liger_ref.rope(q, k, cos, sin)
    th = rp.rotation_thetas(d)
    pos = np.arange(tlen, dtype=np.float64)
    for bi in range(b):
        for h in range(nq):
            np.testing.assert_allclose(qo[bi, h], rp.rope_apply(q[bi, h], th, pos), atol=1e-14)
        for h in range(nk):
            np.testing.assert_allclose(ko[bi, h], rp.rope_apply(k[bi, h], th, pos), atol=1e-14)


def test_glu_port_vs_reference(golden):
    x1, x2, dy = golden["glu_x1"], golden["glu_x2"], golden["glu_dy"]
    np.testing.assert_allclose(rp.swiglu_forward(x1, x2), golden["swiglu_y"], **STRICT)
    a, b = rp.swiglu_backward(dy, x1, x2)
    np.testing.assert_allclose(a, golden["swiglu_dx1"], **STRICT)
    np.testing.assert_allclose(b, golden["swiglu_dx2"], **STRICT)
    np.testing.assert_allclose(rp.geglu_forward(x1, x2), golden["geglu_y"], **STRICT)
    a, b = rp.geglu_backward(dy, x1, x2)
    np.testing.assert_allclose(a, golden["geglu_dx1"], **STRICT)
    np.testing.assert_allclose(b, golden["geglu_dx2"], **STRICT)


def test_chunk_plan_table(golden):
    for bt, v, h, want in golden["plan_table"]:
        assert plan_chunks(int(bt), int(v), int(h)).chunk_rows == want
        assert rp.plan_chunk_rows(int(bt), int(v), int(h)) == want


def test_chunk_plan_validation():
    with pytest.raises(ValueError):
        ChunkPlan(chunk_rows=3, num_chunks=1, total_rows=3, scale_ratio=1.0)
    with pytest.raises(ValueError):
        ChunkPlan(chunk_rows=8, num_chunks=1, total_rows=3, scale_ratio=1.0)
    with pytest.raises(ValueError):
        ChunkPlan(chunk_rows=2, num_chunks=1, total_rows=3, scale_ratio=1.0)
    p = b200_plan(8192, 128256, 4096)  # cfg2: 3 chunks of 11 / 11 / 10 CTA-pair tiles
    assert p.chunk_rows == 2816 and p.num_chunks == 3
    assert b200_plan(7373, 128256, 4096).chunk_rows == 2560  # cfg2's kept rows: 10 / 10 / 9 tiles
    assert b200_plan(1024, 4096, 512).num_chunks == 1
    assert b200_plan(3000, 128256, 4096).num_chunks == 1  # <= 3072 rows: one chunk
    assert (b200_plan(16384, 128256, 4096).chunk_rows, b200_plan(16384, 128256, 4096).num_chunks) == (2816, 6)
    assert b200_plan(65536, 128256, 4096).chunk_rows == 4096  # cfg5 at N = 1: 16 chunks
    assert b200_plan(8192, 256000, 3584).num_chunks == 3  # cfg4: 2816-row chunks, a 1.44 GB buffer
    assert b200_plan(7373, 256000, 3584).chunk_rows == 2560  # cfg4's kept rows
    assert b200_plan(65536, 256000, 3584).chunk_rows == 3072  # the 1.5 GiB buffer caps V = 256000
    assert b200_plan(8192, 128256, 4096, elem_bytes=4).chunk_rows == 2048  # fp32 logits: 1 GiB cap
    for bt in (1, 255, 3073, 9000, 20000, 100000):
        q = b200_plan(bt, 128256, 4096)
        assert q.num_chunks == -(-bt // q.chunk_rows) and (q.chunk_rows % 256 == 0 or q.chunk_rows == bt)


def test_flce_properties_f64():
    x, w, t = cfg1_problem(seed=3, bt=96, h=24, v=70)
    l1, dx1, dw1 = rp.flce_forward_backward(x, w, t, chunk_rows=1)
    l2, dx2, dw2 = rp.flce_forward_backward(x, w, t, chunk_rows=128)
    assert l1 == pytest.approx(l2, rel=1e-12)
    np.testing.assert_allclose(dx1, dx2, atol=1e-15)
    np.testing.assert_allclose(dw1, dw2, atol=1e-14)
    ls, dxs, dws = rp.flce_forward_backward(x, w, t, mean=False)
    assert ls / 96 == pytest.approx(l2, rel=1e-14)
    # dW additive over row groups (pins the token-sharded all-reduce, tests/test_flce.py:182-205)
    _, _, dwa = rp.flce_forward_backward(x[:40], w, t[:40], mean=False)
    _, _, dwb = rp.flce_forward_backward(x[40:], w, t[40:], mean=False)
    np.testing.assert_allclose(dwa + dwb, dws, atol=1e-12)
    # sum over vocab of dW is zero (softmax-minus-onehot rows sum to zero)
    np.testing.assert_allclose(dws.sum(axis=1), 0.0, atol=1e-10)


def test_target_out_of_range_raises():
    with pytest.raises(rp.TargetOutOfRange):
        rp.cross_entropy_(np.zeros((2, 4)), [0, 4])
    with pytest.raises(rp.TargetOutOfRange):
        rp.cross_entropy_(np.zeros((1, 4)), [-100])


def test_liger_ref_token_scaling_matches_liger_formula():
    """use_token_scaling restated per LK/ops/fused_linear_cross_entropy.py:109-139, 187-206 with
    torch-CPU float64: loss_i * p_t (detached), gradient rows scaled alike."""
    import torch

    rng = np.random.default_rng(3)
    z = rng.normal(size=(12, 30)) * 2
    t = rng.integers(0, 30, 12)
    t[4] = -100
    loss, rows, _, g = liger_ref.ce(z, t, reduction="sum", token_scaling=True, label_smoothing=0.1)
    zt = torch.tensor(z, requires_grad=True)
    tt = torch.tensor(t)
    per = torch.nn.functional.cross_entropy(zt, tt, reduction="none", ignore_index=-100, label_smoothing=0.1)
    p = torch.softmax(zt.detach(), -1).gather(1, tt.clamp(min=0)[:, None])[:, 0] * (tt != -100)
    (per * p).sum().backward()
    np.testing.assert_allclose(loss, float((per * p).sum()), rtol=1e-12)
    np.testing.assert_allclose(g, zt.grad.numpy(), rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("ls", [0.0, 0.1])
@pytest.mark.parametrize("reduction", ["mean", "sum", "none"])
def test_liger_ref_class_weights_match_torch(reduction, ls):
    """Class weights (with and without smoothing) restated per LK/ops/cross_entropy.py:122-124,
    165-171, 220-239, 278-288 equal torch-CPU float64 F.cross_entropy(weight=, label_smoothing=)."""
    import torch

    rng = np.random.default_rng(4)
    z = rng.normal(size=(16, 25)) * 2
    t = rng.integers(0, 25, 16)
    t[[3, 9]] = -100
    w = rng.random(25) + 0.2
    loss, _, _, g = liger_ref.ce(z, t, weight=w, reduction=reduction, label_smoothing=ls)
    zt = torch.tensor(z, requires_grad=True)
    ref = torch.nn.functional.cross_entropy(zt, torch.tensor(t), weight=torch.tensor(w), ignore_index=-100,
                                            reduction=reduction, label_smoothing=ls)
    ref.sum().backward()
    np.testing.assert_allclose(loss, ref.detach().numpy(), rtol=1e-12)
    np.testing.assert_allclose(g, zt.grad.numpy(), rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("opts", [dict(), dict(reduction="sum"), dict(reduction="none"), dict(label_smoothing=0.1),
                                  dict(softcap=3.0), dict(softcap=5.0, label_smoothing=0.1, lse_square_scale=1e-3),
                                  dict(bias=True)])
def test_torch_ref_pinned_to_liger_oracle(opts):
    """tests/torch_ref.flce_ref (the checker at full BASELINE sizes, run in fp32 on the GPU) is the
    same math as the pinned float64 oracle: in float64 on CPU it matches liger_ref.flce to
    round-off, chunked and unchunked, so the full-size GPU checks inherit the oracle's pin."""
    import torch

    from tests.torch_ref import flce_ref

    rng = np.random.default_rng(11)
    bt, h, v = 37, 16, 53
    x = rng.uniform(-1, 1, (bt, h))
    w = rng.uniform(-1, 1, (v, h)) * 1.5
    t = rng.integers(0, v, bt)
    t[rng.random(bt) < 0.2] = -100
    kw = dict(opts)
    b = rng.normal(size=v) if kw.pop("bias", False) else None
    ref_loss, ref_rows, _, rgx, rgw, rgb = liger_ref.flce(x, w, t, bias=b, **kw)
    for chunk in (5, 2048):
        loss, rows, gx, gw, gb = flce_ref(torch.tensor(x), torch.tensor(w), torch.tensor(t),
                                          bias=None if b is None else torch.tensor(b), chunk=chunk,
                                          compute_dtype=torch.float64, **kw)
        np.testing.assert_allclose(loss.numpy(), ref_loss, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(rows.numpy(), ref_rows, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(gx.numpy(), rgx, rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(gw.numpy(), rgw, rtol=1e-10, atol=1e-14)
        if b is not None:
            np.testing.assert_allclose(gb.numpy(), rgb, rtol=1e-10, atol=1e-14)
