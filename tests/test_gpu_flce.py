"""Fused linear cross entropy on the GPU (GPU).

* fp32 (SIMT FFMA path) against the reference's own golden vectors at rtol 1e-4;
* bf16 (tcgen05 path) against the float64 oracle evaluated on bf16-rounded inputs at
  rtol 2e-2, with ignore_index / label smoothing / softcap / z-loss / reductions / bias;
* exact ignore masking and non-ignored counts;
* full BASELINE sizes (cfg2 Llama-3-8B head, cfg4 Gemma-2 head) against a cuBLAS fp32
  restatement plus size-independent properties (chunk invariance, determinism,
  sum-over-vocab of dW = 0).
"""

import math

import numpy as np
import pytest
import torch

import paper_2410_10989_b200 as lk
from oracle import liger_ref
from paper_2410_10989_b200 import _capi, errors
from paper_2410_10989_b200.fused_linear_cross_entropy import fused_linear_cross_entropy_forward as flce_fwd
from tests.conftest import rel_close
from tests.torch_ref import close, flce_ref, rel_err

pytestmark = pytest.mark.gpu


def cuda(a, dtype=torch.float32):
    return torch.tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def flce(x, w, t, **kw):
    loss, z, _, _, gx, gw, gb = flce_fwd(x, w, t, compute_grad_input=True, compute_grad_weight=True, **kw)
    torch.cuda.synchronize()
    return loss, z, gx, gw, gb


# ------------------------------------------------------------- fp32 vs golden
@pytest.mark.parametrize("chunk", [1, 8, 64])
def test_fp32_small_vs_reference_golden(golden, chunk):
    x = cuda(golden["flce_small_x"])
    w = cuda(golden["flce_small_w_hv"].T)
    t = cuda(golden["flce_small_t"], torch.long)
    loss, _, gx, gw, _ = flce(x, w, t, chunk_rows=chunk)
    assert loss.item() == pytest.approx(float(golden[f"flce_small_c{chunk}_loss"]), rel=1e-4)
    for got, ref in ((gx, golden[f"flce_small_c{chunk}_dx"]), (gw, golden[f"flce_small_c{chunk}_dw_hv"].T)):
        ok, err = rel_close(got.cpu().numpy(), ref, 1e-4)
        assert ok, err


def test_fp32_mid_scalar_and_cfg1_vs_reference_golden(golden):
    for name in ("mid", "scalar"):
        x = cuda(golden[f"flce_{name}_x"])
        w = cuda(golden[f"flce_{name}_w_hv"].T)
        t = cuda(golden[f"flce_{name}_t"], torch.long)
        loss, _, gx, gw, _ = flce(x, w, t)
        assert loss.item() == pytest.approx(float(golden[f"flce_{name}_loss"]), rel=1e-4)
        assert rel_close(gx.cpu().numpy(), golden[f"flce_{name}_dx"], 1e-4)[0]
        assert rel_close(gw.cpu().numpy(), golden[f"flce_{name}_dw_hv"].T, 1e-4)[0]
    # cfg1: BT=1024, H=512, V=4096, f32, seed 0
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (1024, 512))
    w_hv = rng.uniform(-1, 1, (512, 4096)) / math.sqrt(512)
    t = rng.integers(0, 4096, 1024)
    loss, _, gx, gw, _ = flce(cuda(x), cuda(w_hv.T), cuda(t, torch.long))
    assert loss.item() == pytest.approx(float(golden["flce_cfg1_loss"]), rel=1e-4)
    dx = gx.double().cpu().numpy()
    dw_hv = gw.double().cpu().numpy().T
    assert rel_close(dx.reshape(-1)[golden["flce_cfg1_dx_idx"]], golden["flce_cfg1_dx_val"], 1e-4)[0]
    assert rel_close(dw_hv.reshape(-1)[golden["flce_cfg1_dw_hv_idx"]], golden["flce_cfg1_dw_hv_val"], 1e-4)[0]
    assert np.abs(dw_hv).sum() == pytest.approx(float(golden["flce_cfg1_dw_abssum"]), rel=1e-4)
    assert np.abs(dx).sum() == pytest.approx(float(golden["flce_cfg1_dx_abssum"]), rel=1e-4)


# ------------------------------------------------------ bf16 vs f64 oracle
def bf16_problem(bt, h, v, seed, ignore_frac=0.1, wscale=1.0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (bt, h))
    w = rng.uniform(-1, 1, (v, h)) / math.sqrt(h) * wscale
    t = rng.integers(0, v, bt)
    t[rng.random(bt) < ignore_frac] = -100
    xb = cuda(x, torch.bfloat16)
    wb = cuda(w, torch.bfloat16)
    return xb, wb, cuda(t, torch.long), xb.double().cpu().numpy(), wb.double().cpu().numpy(), t


@pytest.mark.parametrize(
    "opts",
    [
        dict(),
        dict(reduction="sum"),
        dict(label_smoothing=0.1),
        dict(softcap=30.0),
        dict(softcap=5.0, label_smoothing=0.1, lse_square_scale=1e-4),
        dict(chunk_rows=128),
        dict(chunk_rows=384),
    ],
)
def test_bf16_cfg1_shape_vs_oracle(opts):
    xb, wb, tb, x, w, t = bf16_problem(1024, 512, 4096, seed=1, wscale=4.0)
    kw = {k: v for k, v in opts.items() if k != "chunk_rows"}
    loss, _, gx, gw, _ = flce(xb, wb, tb, **opts)
    ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(x, w, t, **kw)
    assert rel_close(loss.item(), ref_loss, 2e-2)[0]
    ok, err = rel_close(gx.float().cpu().numpy(), rgx, 2e-2)
    assert ok, ("dx", err)
    ok, err = rel_close(gw.float().cpu().numpy(), rgw, 2e-2)
    assert ok, ("dw", err)
    assert torch.all(gx[tb == -100] == 0)


def test_bf16_ragged_shapes_and_bias():
    # H % 64 != 0, V % 256 != 0, BT not a multiple of the chunk
    xb, wb, tb, x, w, t = bf16_problem(333, 200, 1000, seed=2)
    bias = torch.randn(1000, device="cuda").to(torch.bfloat16)
    loss, _, gx, gw, gb = flce(xb, wb, tb, bias=bias, chunk_rows=128)
    ref_loss, _, _, rgx, rgw, rgb = liger_ref.flce(x, w, t, bias=bias.double().cpu().numpy())
    assert rel_close(loss.item(), ref_loss, 2e-2)[0]
    assert rel_close(gx.float().cpu().numpy(), rgx, 2e-2)[0]
    assert rel_close(gw.float().cpu().numpy(), rgw, 2e-2)[0]
    assert rel_close(gb.float().cpu().numpy(), rgb, 2e-2)[0]


@pytest.mark.parametrize("kw", [dict(), dict(label_smoothing=0.1, softcap=30.0), dict(softcap=5.0),
                                dict(lse_square_scale=1e-4, reduction="sum")])
@pytest.mark.parametrize("env", ["finalize_block", "separate_cast"])
def test_ring_finalize_and_folded_dw_cast_match_reference_paths(kw, env):
    """Default path (TMA-ring finalize, dW cast folded into the last chunk's epilogue) vs the
    one-CTA-per-row finalize / separate cast kernel, and the oracle."""
    xb, wb, tb, x, w, t = bf16_problem(1000, 256, 4096, seed=11)
    if env == "separate_cast":
        kw = dict(kw, accum_dtype=torch.float32)  # the fold only exists on the fp32-accumulator path
    a = flce(xb, wb, tb, chunk_rows=256, **kw)
    knob = _capi.PATH_FLCE_FINALIZE if env == "finalize_block" else _capi.PATH_FLCE_SEPARATE_CAST
    with _capi.select_path(knob, 1):
        b = flce(xb, wb, tb, chunk_rows=256, **kw)
    assert rel_err(a[0], b[0]) < 1e-5
    assert close(a[2], b[2], 1e-2) and close(a[3], b[3], 1e-2)
    ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(x, w, t, **{k: v for k, v in kw.items() if k != "accum_dtype"})
    assert rel_close(a[0].item(), ref_loss, 2e-2)[0]
    ok, err = rel_close(a[2].float().cpu().numpy(), rgx, 2e-2)
    assert ok, err
    ok, err = rel_close(a[3].float().cpu().numpy(), rgw, 2e-2)
    assert ok, err
    assert torch.all(a[2][tb == -100] == 0)


@pytest.mark.parametrize("accum_dtype", [None, torch.float32, torch.bfloat16])
@pytest.mark.parametrize("chunk", [256, 64])  # 4 and 16 chunks (auto: bf16 / fp32 accumulation)
def test_grad_weight_accumulation_modes(accum_dtype, chunk):
    """Liger's accum_dtype (LK/ops/fused_linear_cross_entropy.py:64-69): fp32 workspace or a
    weight-dtype TMA reduce-add across chunks; all within the bf16 tolerance of the oracle."""
    xb, wb, tb, x, w, t = bf16_problem(1000, 256, 4096, seed=12)
    loss, _, gx, gw, _ = flce(xb, wb, tb, chunk_rows=chunk, accum_dtype=accum_dtype)
    ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(x, w, t)
    assert rel_close(loss.item(), ref_loss, 2e-2)[0]
    ok, err = rel_close(gx.float().cpu().numpy(), rgx, 2e-2)
    assert ok, err
    ok, err = rel_close(gw.float().cpu().numpy(), rgw, 2e-2)
    assert ok, err
    if accum_dtype == torch.float32:  # tighter: fp32 accumulation over chunks
        ok, err = rel_close(gw.float().cpu().numpy(), rgw, 1e-2)
        assert ok, err


def test_tcgen05_matches_simt_path():
    xb, wb, tb, *_ = bf16_problem(512, 256, 2048, seed=3)
    a = flce(xb, wb, tb, chunk_rows=256)
    b = flce(xb, wb, tb, chunk_rows=256, force_simt=True)
    assert rel_err(a[0], b[0]) < 1e-3
    assert close(a[2], b[2], 2e-2) and close(a[3], b[3], 2e-2)


def test_reduction_none_and_module_backward():
    xb, wb, tb, x, w, t = bf16_problem(256, 128, 1024, seed=4)
    xr = xb.clone().requires_grad_(True)
    wr = wb.clone().requires_grad_(True)
    loss = lk.LigerFusedLinearCrossEntropyLoss(reduction="none")(wr, xr, tb)
    assert loss.shape == (256,) and loss.dtype == torch.float32
    loss.sum().backward()
    _, rrows, _, rgx, rgw, _ = liger_ref.flce(x, w, t, reduction="none")
    assert rel_close(loss.detach().cpu().numpy(), rrows, 2e-2)[0]
    assert rel_close(xr.grad.float().cpu().numpy(), rgx, 2e-2)[0]
    # mean loss scaled by 2 through autograd
    xr.grad = None
    wr.grad = None
    (2.0 * lk.LigerFusedLinearCrossEntropyLoss()(wr, xr, tb)).backward()
    ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(x, w, t)
    assert rel_close(xr.grad.float().cpu().numpy(), 2 * rgx, 2e-2)[0]
    assert rel_close(wr.grad.float().cpu().numpy(), 2 * rgw, 2e-2)[0]


def test_exact_ignore_masking_and_counts():
    xb, wb, tb, *_ = bf16_problem(777, 128, 3000, seed=5, ignore_frac=0.3)
    loss, _, _, _, gx, gw, _ = flce_fwd(xb, wb, tb, reduction="none", compute_grad_input=True,
                                       compute_grad_weight=True)
    ign = tb == -100
    assert torch.all(loss[ign] == 0) and torch.all(gx[ign] == 0)
    assert torch.all(loss[~ign] > 0)
    # count used for MEAN equals the exact integer count
    mean = flce_fwd(xb, wb, tb, reduction="mean")[0]
    ssum = flce_fwd(xb, wb, tb, reduction="sum")[0]
    n = int((~ign).sum())
    assert mean.item() == pytest.approx(ssum.item() / n, rel=1e-6)
    all_ign = torch.full_like(tb, -100)
    l0, _, _, _, g0, w0, _ = flce_fwd(xb, wb, all_ign, compute_grad_input=True, compute_grad_weight=True)
    assert l0.item() == 0.0 and torch.all(g0 == 0) and torch.all(w0 == 0)


def test_target_out_of_range_raises():
    xb, wb, tb, *_ = bf16_problem(64, 64, 128, seed=6, ignore_frac=0.0)
    tb[3] = 128
    with pytest.raises(errors.TargetOutOfRange):
        flce_fwd(xb, wb, tb)


@pytest.mark.parametrize("bad", [128, 100000, -5])
def test_target_out_of_range_with_class_weights_raises(bad):
    """Class weights are indexed by target: an out-of-range target must raise the typed error,
    not read past the weight vector."""
    xb, wb, tb, *_ = bf16_problem(64, 64, 128, seed=6, ignore_frac=0.0)
    tb[3] = bad
    cw = torch.rand(128, device="cuda") + 0.5
    with pytest.raises(errors.TargetOutOfRange):
        flce_fwd(xb, wb, tb, ce_weight=cw)
    with pytest.raises(errors.TargetOutOfRange):
        flce_fwd(xb, wb, tb, ce_weight=cw, label_smoothing=0.1)
    x = torch.randn(8, 128, device="cuda")
    t = torch.randint(0, 128, (8,), device="cuda")
    t[2] = bad
    with pytest.raises(errors.TargetOutOfRange):
        lk.LigerCrossEntropyLoss(weight=cw)(x, t)
    torch.cuda.synchronize()  # no illegal-address fault left behind


def test_no_grad_forward_matches():
    xb, wb, tb, x, w, t = bf16_problem(300, 64, 700, seed=8)
    loss = flce_fwd(xb, wb, tb, compute_grad_input=False)[0]
    assert rel_close(loss.item(), liger_ref.flce(x, w, t)[0], 2e-2)[0]


# -------------------------------------------------------- full BASELINE sizes
def big_problem(bt, h, v, seed, wscale=1.0, ignore_frac=0.1):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.rand(bt, h, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(v, h, device="cuda", generator=g) * 2 - 1) * (wscale / 64.0)).to(torch.bfloat16)
    t = torch.randint(0, v, (bt,), device="cuda", generator=g)
    t[torch.rand(bt, device="cuda", generator=g) < ignore_frac] = -100
    return x, w, t


def test_cfg5_one_gpu_default_plan():
    """BASELINE configs[4] on one GPU: 65536 tokens of the Llama-3-8B head.  The default plan
    takes 4096-row chunks above 16384 tokens (16 chunks, so grad_w accumulates in the fp32
    workspace); checked against the chunked fp32 restatement (pinned to the oracle), the
    2048-row plan, and a second run (bitwise)."""
    x, w, t = big_problem(65536, 4096, 128256, seed=2)
    assert lk.flce_plan(65536, 4096, 128256) == (4096, 16)
    loss, _, gx, gw, _ = flce(x, w, t)
    rloss, _, rgx, rgw, _ = flce_ref(x, w, t, chunk=4096)
    assert abs(loss.item() - rloss.item()) <= 2e-2 * abs(rloss.item())
    assert close(gx, rgx, 2e-2), rel_err(gx, rgx)
    assert close(gw, rgw, 2e-2), rel_err(gw, rgw)
    assert torch.all(gx[t == -100] == 0)
    del rgx, rgw
    loss2, _, gx2, gw2, _ = flce(x, w, t)
    assert loss.item() == loss2.item() and torch.equal(gx, gx2) and torch.equal(gw, gw2)
    del gx2, gw2
    loss3, _, gx3, gw3, _ = flce(x, w, t, chunk_rows=2048)
    assert abs(loss3.item() - loss.item()) <= 1e-4 * abs(loss.item())
    assert close(gx3, gx, 1e-2) and close(gw3, gw, 2e-2)


def test_finalize_ring_bitwise_repeatable():
    """The FLCE finalize (CE ring, one HBM pass) releases each ring stage only after its shared-
    memory loads have returned (ring::release_after_loads).  With a plain arrive, ~1 in 5 calls
    of this shape differed in one 256-column stretch of one row (the producer's refill overwrote
    the stage under late loads; profiles/r02/ring_release_race.md).  Gemma-2 head width, one
    2048-row chunk, softcap + smoothing, 12 calls: all bitwise equal."""
    x, w, t = big_problem(2048, 3584, 256000, seed=1, wscale=30.0)
    kw = dict(softcap=30.0, label_smoothing=0.1, chunk_rows=2048)
    loss0, _, _, _, gx0, _, _ = flce_fwd(x, w, t, compute_grad_input=True, compute_grad_weight=False,
                                         reduction="none", **kw)
    for _ in range(11):
        loss, _, _, _, gx, _, _ = flce_fwd(x, w, t, compute_grad_input=True, compute_grad_weight=False,
                                           reduction="none", **kw)
        assert torch.equal(loss, loss0) and torch.equal(gx, gx0)


def test_cfg2_llama3_head_vs_torch_fp32_and_properties():
    x, w, t = big_problem(8192, 4096, 128256, seed=0)
    loss, _, gx, gw, _ = flce(x, w, t)
    rloss, _, rgx, rgw, _ = flce_ref(x, w, t)
    assert abs(loss.item() - rloss.item()) <= 2e-2 * abs(rloss.item())
    assert close(gx, rgx, 2e-2), rel_err(gx, rgx)
    assert close(gw, rgw, 2e-2), rel_err(gw, rgw)
    rgw_keep = rgw
    del rgx
    assert torch.all(gx[t == -100] == 0)
    # sum over the vocabulary of dW vanishes (softmax - onehot rows sum to zero) up to the
    # bf16 rounding of dlogits and of grad_w; the default accumulates grad_w in bf16 across
    # the 4 chunks exactly in Liger's order (acc = bf16(acc + bf16(chunk product)),
    # LK/ops/fused_linear_cross_entropy.py:211), which doubles that noise vs fp32 accumulation
    colsum = gw.float().sum(0)
    assert colsum.abs().max().item() < 2e-2 * gw.float().abs().max().item() * 128
    # fp32 accumulation across chunks: one final rounding, tighter against the fp32 reference
    _, _, _, gw32, _ = flce(x, w, t, accum_dtype=torch.float32)
    assert close(gw32, rgw_keep, 1e-2)
    colsum32 = gw32.float().sum(0)
    assert colsum32.abs().max().item() < 2e-2 * gw32.float().abs().max().item() * 64
    del gw32
    # determinism: bitwise identical on a second run
    loss2, _, gx2, gw2, _ = flce(x, w, t)
    assert loss.item() == loss2.item() and torch.equal(gx, gx2) and torch.equal(gw, gw2)
    # chunk-schedule invariance (reference plan, 32 chunks of 256 rows)
    loss3, _, gx3, gw3, _ = flce(x, w, t, chunk_rows=256)
    assert abs(loss3.item() - loss.item()) <= 1e-4 * abs(loss.item())
    assert close(gx3, gx, 1e-2) and close(gw3, gw, 2e-2)


def test_cfg4_gemma2_head_softcap_smoothing():
    # Gemma-2-9B head: H=3584, V=256000, softcap 30, label smoothing 0.1 (stress scale: logit sigma ~ 10)
    # BT = 8192: 8192 x 256000 logits = 2.1e9 elements, above 2^31 - 1 bytes in
    # bf16, in 4 chunks; flce_ref is pinned to oracle.liger_ref (tests/test_oracle.py)
    x, w, t = big_problem(8192, 3584, 256000, seed=1, wscale=30.0)
    kw = dict(softcap=30.0, label_smoothing=0.1)
    loss, _, gx, gw, _ = flce(x, w, t, **kw)
    rloss, _, rgx, rgw, _ = flce_ref(x, w, t, **kw)
    assert abs(loss.item() - rloss.item()) <= 2e-2 * abs(rloss.item())
    assert close(gx, rgx, 2e-2), rel_err(gx, rgx)
    assert close(gw, rgw, 2e-2), rel_err(gw, rgw)
    assert torch.all(gx[t == -100] == 0)
    del rgx, rgw
    loss2, _, gx2, gw2, _ = flce(x, w, t, **kw)  # bitwise deterministic
    assert loss.item() == loss2.item() and torch.equal(gx, gx2) and torch.equal(gw, gw2)


@pytest.mark.parametrize("path", ["bf16", "fp32_simt", "fp32_tc"])
@pytest.mark.parametrize("kw", [dict(), dict(softcap=30.0, label_smoothing=0.1)])
def test_flce_token_accuracy_and_predicted_tokens(path, kw):
    """Liger return_token_accuracy / return_predicted_tokens on the FLCE head (argmax of the rounded,
    softcapped logits; the tcgen05 paths track it in the logits epilogue, no extra pass)."""
    xb, wb, tb, x, w, t = bf16_problem(700, 256, 5000, seed=21)
    simt = path == "fp32_simt"
    if path != "bf16":
        xb, wb = xb.float(), wb.float()
    logits = xb.float() @ wb.float().T
    if "softcap" in kw:
        logits = kw["softcap"] * torch.tanh(logits / kw["softcap"])
    logits = logits.to(xb.dtype).float()
    tb = tb.clone()
    tb[::4] = logits[::4].argmax(1)
    tb[::9] = -100
    loss, _, acc, pred, gx, gw, _ = flce_fwd(xb, wb, tb, compute_grad_input=True, compute_grad_weight=True,
                                              return_token_accuracy=True, return_predicted_tokens=True,
                                              force_simt=simt, chunk_rows=256, **kw)
    ign = tb == -100
    want = logits.argmax(1)
    want[ign] = -1
    assert torch.all(pred[ign] == -1)
    agree = (pred == want).float().mean().item()
    assert agree > 0.99, agree
    mism = (pred != want) & ~ign
    if mism.any():  # GEMM summation order: a disagreement is a near-tie of the rounded logits
        r = mism.nonzero().flatten()
        gap = (logits[r, want[r]] - logits[r, pred[r]]).abs()
        assert torch.all(gap <= 2 ** -7 * logits[r, want[r]].abs() + 1e-6)
    correct = ((pred == tb) & ~ign).float()
    assert abs(acc.item() - correct.sum().item() / (~ign).sum().item()) < 1e-6
    loss2, _, _, _, gx2, gw2, _ = flce_fwd(xb, wb, tb, compute_grad_input=True, compute_grad_weight=True,
                                           force_simt=simt, chunk_rows=256, **kw)
    assert loss.item() == loss2.item() and torch.equal(gx, gx2) and torch.equal(gw, gw2)


@pytest.mark.parametrize("accum_dtype", [None, torch.float32])
@pytest.mark.parametrize("slices", [2, 4, 5])
def test_grad_w_slices_with_events_bitwise(slices, accum_dtype):
    """Token-sharded overlap hook: the last chunk's grad_w GEMM in vocab-row slices with one
    event per slice gives bitwise the same gradients (same tiles, same K order)."""
    xb, wb, tb, *_ = bf16_problem(1000, 256, 5000, seed=31)
    a = flce(xb, wb, tb, chunk_rows=256, accum_dtype=accum_dtype)
    events = [torch.cuda.Event() for _ in range(slices)]
    b_loss, _, _, _, b_gx, b_gw, _ = flce_fwd(xb, wb, tb, compute_grad_input=True, compute_grad_weight=True,
                                              chunk_rows=256, accum_dtype=accum_dtype, grad_w_slice_events=events)
    for ev in events:
        ev.synchronize()
    torch.cuda.synchronize()
    assert a[0].item() == b_loss.item()
    assert torch.equal(a[2], b_gx) and torch.equal(a[3], b_gw)


@pytest.mark.parametrize("slices", [2, 5])
def test_fp32_grad_w_slices_with_events_bitwise(slices):
    """The same hook on the fp32 split-operand path: each slice re-addresses the dZ pieces at a
    vocab-row offset (piece-major layout, Problem::kb_term runs), bitwise equal to one launch."""
    g = torch.Generator(device="cuda").manual_seed(32)
    x = torch.rand(700, 256, device="cuda", generator=g) * 2 - 1
    w = (torch.rand(3000, 256, device="cuda", generator=g) * 2 - 1) / 16
    t = torch.randint(0, 3000, (700,), device="cuda", generator=g)
    a = flce(x, w, t, chunk_rows=300)
    events = [torch.cuda.Event() for _ in range(slices)]
    b_loss, _, _, _, b_gx, b_gw, _ = flce_fwd(x, w, t, compute_grad_input=True, compute_grad_weight=True,
                                              chunk_rows=300, grad_w_slice_events=events)
    torch.cuda.synchronize()
    assert a[0].item() == b_loss.item()
    assert torch.equal(a[2], b_gx) and torch.equal(a[3], b_gw)


@pytest.mark.parametrize("shape", [(1, 8, 5), (3, 16, 77), (65, 72, 130), (129, 64, 4096)])
def test_fp32_split_path_tiny_and_ragged_shapes(shape):
    """fp32 split-operand path at the edges of its K runs: one row, H = 8 (a run of one partial
    k-block), V below and across the 64-column padding, chunk rows not a multiple of 64 --
    against the float64 oracle at the fp32 tolerance."""
    bt, h, v = shape
    rng = np.random.default_rng(bt * 7 + h)
    x = rng.uniform(-1, 1, (bt, h)).astype(np.float32)
    w = (rng.uniform(-1, 1, (v, h)) / math.sqrt(h)).astype(np.float32)
    t = rng.integers(0, v, bt)
    ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(x.astype(np.float64), w.astype(np.float64), t)
    loss, _, gx, gw, _ = flce(cuda(x), cuda(w), cuda(t, torch.long), chunk_rows=max(1, bt // 2))
    assert loss.item() == pytest.approx(ref_loss, rel=1e-4)
    assert rel_close(gx.double().cpu().numpy(), rgx, 1e-4)[0]
    assert rel_close(gw.double().cpu().numpy(), rgw, 1e-4)[0]


@pytest.mark.parametrize("simt", [False, True])
@pytest.mark.parametrize("kw", [dict(), dict(label_smoothing=0.1, softcap=30.0, lse_square_scale=1e-4)])
def test_flce_use_token_scaling(simt, kw):
    """Liger use_token_scaling (LK/ops/fused_linear_cross_entropy.py:109-139, 187-206): loss and
    gradients of each row scaled by its detached target probability, vs the float64 oracle."""
    xb, wb, tb, x, w, t = bf16_problem(600, 128, 3000, seed=41, wscale=4.0)
    if simt:
        xb, wb = xb.float(), wb.float()
        x, w = xb.double().cpu().numpy(), wb.double().cpu().numpy()
    loss, _, _, _, gx, gw, _ = flce_fwd(xb, wb, tb, compute_grad_input=True, compute_grad_weight=True,
                                        use_token_scaling=True, force_simt=simt, chunk_rows=256, **kw)
    ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(x, w, t, token_scaling=True, **kw)
    tol = 1e-4 if simt else 2e-2
    assert rel_close(loss.item(), ref_loss, tol)[0], (loss.item(), ref_loss)
    ok, err = rel_close(gx.float().cpu().numpy(), rgx, tol)
    assert ok, err
    ok, err = rel_close(gw.float().cpu().numpy(), rgw, tol)
    assert ok, err


@pytest.mark.parametrize("kw", [dict(), dict(label_smoothing=0.1), dict(label_smoothing=0.1, softcap=30.0)])
@pytest.mark.parametrize("simt", [False, True])
@pytest.mark.parametrize("reduction", ["mean", "sum"])
def test_flce_ce_weight(simt, reduction, kw):
    """Liger ce_weight on the FLCE head (with and without label smoothing) vs the float64 oracle."""
    xb, wb, tb, x, w, t = bf16_problem(700, 128, 3000, seed=43, wscale=3.0)
    if simt:
        xb, wb = xb.float(), wb.float()
        x, w = xb.double().cpu().numpy(), wb.double().cpu().numpy()
    cw = torch.rand(3000, device="cuda") + 0.2
    loss, _, _, _, gx, gw, _ = flce_fwd(xb, wb, tb, cw, compute_grad_input=True, compute_grad_weight=True,
                                        reduction=reduction, force_simt=simt, chunk_rows=256, lse_square_scale=1e-4,
                                        **kw)
    ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(x, w, t, weight=cw.double().cpu().numpy(), reduction=reduction,
                                                 lse_square_scale=1e-4, **kw)
    tol = 1e-4 if simt else 2e-2
    assert rel_close(loss.item(), ref_loss, tol)[0], (loss.item(), ref_loss)
    ok, err = rel_close(gx.float().cpu().numpy(), rgx, tol)
    assert ok, err
    ok, err = rel_close(gw.float().cpu().numpy(), rgw, tol)
    assert ok, err


@pytest.mark.parametrize("kw", [dict(), dict(label_smoothing=0.1, softcap=30.0)])
def test_fp16_tcgen05_path_vs_oracle(kw):
    """fp16 operands through the tcgen05 path (kind::f16 with the f16 descriptor format)."""
    rng = np.random.default_rng(51)
    bt, h, v = 700, 256, 3000
    x = rng.uniform(-1, 1, (bt, h))
    w = rng.uniform(-1, 1, (v, h)) / math.sqrt(h) * 3
    t = rng.integers(0, v, bt)
    t[rng.random(bt) < 0.1] = -100
    xh, wh = cuda(x, torch.float16), cuda(w, torch.float16)
    loss, _, gx, gw, _ = flce(xh, wh, cuda(t, torch.long), chunk_rows=256, **kw)
    ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(xh.double().cpu().numpy(), wh.double().cpu().numpy(), t, **kw)
    assert rel_close(loss.item(), ref_loss, 2e-2)[0]
    ok, err = rel_close(gx.float().cpu().numpy(), rgx, 2e-2)
    assert ok, err
    ok, err = rel_close(gw.float().cpu().numpy(), rgw, 2e-2)
    assert ok, err


def test_flce_in_cuda_graph(monkeypatch):
    """No host syncs on the FLCE path: forward + backward capture into a CUDA graph and replay
    to the same bits as eager (counts and the MEAN scale stay on the device).  Under capture
    the ignored rows are skipped with the kept-row count kept on the device
    (KEPT_ROWS_DEVICE_COUNT), so the eager reference runs that mode too; the host-count mode
    matches it to tolerance below."""
    import paper_2410_10989_b200.fused_linear_cross_entropy as flce_mod

    monkeypatch.setattr(flce_mod, "KEPT_ROWS_DEVICE_COUNT", True)
    bt, h, v = 1024, 1024, 16384
    g = torch.Generator(device="cuda").manual_seed(5)
    x = ((torch.rand(bt, h, device="cuda", generator=g) * 2 - 1)).to(torch.bfloat16)
    w = ((torch.rand(v, h, device="cuda", generator=g) * 2 - 1) / 32).to(torch.bfloat16)
    t = torch.randint(0, v, (bt,), device="cuda", generator=g)
    t[::7] = -100
    xs, ws = x.clone().requires_grad_(True), w.clone().requires_grad_(True)
    loss_fn = lk.LigerFusedLinearCrossEntropyLoss()

    def step():
        xs.grad = ws.grad = None
        loss = loss_fn(ws, xs, t)
        loss.backward()
        return loss.detach().clone(), xs.grad.clone(), ws.grad.clone()

    eager = step()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = step()
    graph.replay()
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(eager, out))
    monkeypatch.setattr(flce_mod, "KEPT_ROWS_DEVICE_COUNT", False)
    skipped = step()  # 147 of 1024 rows ignored: the host-count kept-row path
    assert abs(skipped[0].item() - eager[0].item()) <= 1e-3 * abs(eager[0].item())
    assert torch.equal(skipped[1][t == -100], torch.zeros_like(skipped[1][t == -100]))
    assert close(skipped[1], eager[1], 1e-2) and close(skipped[2], eager[2], 2e-2)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_operands_on_different_devices_raise():
    x = torch.randn(8, 64, device="cuda:0", dtype=torch.bfloat16)
    w = torch.randn(128, 64, device="cuda:1", dtype=torch.bfloat16)
    t = torch.randint(0, 128, (8,), device="cuda:0")
    with pytest.raises(errors.ShapeMismatch):
        flce_fwd(x, w, t)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_single_cta_gemm_path_matches_pair(path_knob, dtype):
    """The single-CTA tcgen05 kernel (test knob) with the same operand load modes as the CTA
    pair -- including the piece-addressed fp32 modes 3-5 -- gives the same FLCE results."""
    g = torch.Generator(device="cuda").manual_seed(41)
    x = (torch.rand(300, 264, device="cuda", generator=g) * 2 - 1).to(dtype)
    w = ((torch.rand(2000, 264, device="cuda", generator=g) * 2 - 1) / 16).to(dtype)
    t = torch.randint(0, 2000, (300,), device="cuda", generator=g)
    ref = flce(x, w, t, chunk_rows=128)
    path_knob(_capi.PATH_CTA_GROUP, 1)
    one = flce(x, w, t, chunk_rows=128)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    assert abs(one[0].item() - ref[0].item()) <= tol * abs(ref[0].item())
    assert close(one[2], ref[2], tol) and close(one[3], ref[3], tol)


def _random_flce_cases(n=40, seed=2024):
    """Seeded random FLCE configurations over the option space and the shape edges."""
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        dtype = [torch.float32, torch.bfloat16, torch.float16][i % 3]
        bt = int(rng.choice([1, 7, 64, 130, 333, 700]))
        h = int(rng.choice([8, 24, 64, 136, 256, 520]))
        v = int(rng.choice([5, 63, 257, 1000, 4099]))
        opts = {}
        if rng.random() < 0.4:
            opts["label_smoothing"] = float(rng.choice([0.05, 0.1, 0.3]))
        if rng.random() < 0.3:
            opts["softcap"] = float(rng.choice([5.0, 30.0]))
        if rng.random() < 0.2:
            opts["lse_square_scale"] = 1e-3
        opts["reduction"] = str(rng.choice(["mean", "sum", "none"]))
        chunk = int(rng.choice([0, 1, 32, 100, 256]))
        cases.append((i, dtype, bt, h, v, opts, chunk, bool(rng.random() < 0.25), float(rng.choice([0.0, 0.1, 0.5]))))
    return cases


@pytest.mark.parametrize("case", _random_flce_cases(), ids=lambda c: f"c{c[0]}")
def test_flce_random_configs_vs_oracle(case):
    """40 seeded random configurations (fp32 / bf16 / fp16; 1..700 rows; H from 8 (one partial
    k-block) to 520; V from 5 to 4099; smoothing, softcap, z-loss, bias, all reductions,
    chunk sizes 1..256 and the default; 0-50% ignored targets) against the float64 oracle at
    the north-star tolerance of the dtype, with ignored rows exactly zero."""
    i, dtype, bt, h, v, opts, chunk, use_bias, ign = case
    rng = np.random.default_rng(1000 + i)
    x = rng.uniform(-1, 1, (bt, h))
    w = rng.uniform(-1, 1, (v, h)) / math.sqrt(h) * 3
    b = rng.normal(size=v) * 0.5 if use_bias else None
    t = rng.integers(0, v, bt)
    t[rng.random(bt) < ign] = -100
    xd = torch.tensor(x, dtype=dtype, device="cuda")
    wd = torch.tensor(w, dtype=dtype, device="cuda")
    bd = torch.tensor(b, dtype=dtype, device="cuda") if b is not None else None
    td = torch.tensor(t, device="cuda")
    ref = liger_ref.flce(xd.double().cpu().numpy(), wd.double().cpu().numpy(), t,
                         bias=None if bd is None else bd.double().cpu().numpy(), **opts)
    loss, _, _, _, gx, gw, gb = flce_fwd(xd, wd, td, bias=bd, compute_grad_input=True, compute_grad_weight=True,
                                         chunk_rows=chunk or None, **opts)
    torch.cuda.synchronize()
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    if opts["reduction"] == "none":
        assert rel_close(loss.double().cpu().numpy(), ref[1], tol)[0]
    else:
        assert loss.item() == pytest.approx(ref[0], rel=tol, abs=tol * 1e-3)
    assert rel_close(gx.double().cpu().numpy(), ref[3], tol)[0], "grad_x"
    assert rel_close(gw.double().cpu().numpy(), ref[4], tol)[0], "grad_w"
    if bd is not None:
        assert rel_close(gb.double().cpu().numpy(), ref[5], tol)[0], "grad_bias"
    ignored = torch.tensor(t == -100, device="cuda")
    assert torch.all(gx[ignored] == 0)


@pytest.mark.parametrize("reg", [0, 1])
def test_weight_dtype_accumulation_paths_vs_oracle(reg, path_knob):
    """16-bit grad_w accumulated across 4 chunks: TMA reduce-add in L2 (default) or the
    register read-add-round epilogue (LK_PATH_DW_ACCUM16 = 1), both against the f64 oracle."""
    path_knob(_capi.PATH_DW_ACCUM16, reg)
    xb, wb, tb, x, w, t = bf16_problem(1000, 256, 3000, seed=41)
    loss, _, gx, gw, _ = flce(xb, wb, tb, chunk_rows=256, accum_dtype=torch.bfloat16)
    rl, _, _, rgx, rgw, _ = liger_ref.flce(x, w, t)
    assert rel_close(loss.item(), rl, 2e-2)[0]
    assert rel_close(gx.double().cpu().numpy(), rgx, 2e-2)[0]
    assert rel_close(gw.double().cpu().numpy(), rgw, 2e-2)[0]
