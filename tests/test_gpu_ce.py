"""Standalone cross entropy on the GPU against the CPU oracle (GPU).

fp32: rtol 1e-4 (atol 1e-4 * max|ref|); bf16: rtol 2e-2 (atol 2e-2 * max|ref|)
with the oracle evaluated on the bf16-rounded inputs.  Ignored
rows and token counts are checked exactly.
"""

import numpy as np
import pytest
import torch

import paper_2410_10989_b200 as lk
from oracle import liger_ref, rowfuse_port as rp
from paper_2410_10989_b200 import _capi, errors
from tests.conftest import rel_close

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def run_ce(x_np, t_np, dtype, **kw):
    x = torch.tensor(x_np, dtype=dtype, device="cuda").requires_grad_(True)
    t = torch.tensor(t_np, dtype=torch.long, device="cuda")
    loss_fn = lk.LigerCrossEntropyLoss(**kw)
    loss = loss_fn(x, t)
    if kw.get("reduction", "mean") == "none":
        loss.sum().backward()
    else:
        loss.backward()
    return loss.detach().float().cpu().numpy(), x.grad.float().cpu().numpy()


def test_ce_known_answers(golden):
    for k in (1, 2):
        loss, grad = run_ce(golden[f"ce_kat_{k}_logits"], golden[f"ce_kat_{k}_target"], torch.float32,
                            reduction="sum")
        assert float(loss) == pytest.approx(float(golden[f"ce_kat_{k}_loss"]), rel=1e-5)
        np.testing.assert_allclose(grad, golden[f"ce_kat_{k}_grad"], atol=1e-6)


@pytest.mark.parametrize("case", ["a", "b", "c"])
def test_ce_golden_fp32(golden, case):
    mean = bool(golden[f"ce_rand_{case}_mean"])
    loss, grad = run_ce(golden[f"ce_rand_{case}_logits"], golden[f"ce_rand_{case}_target"], torch.float32,
                        reduction="mean" if mean else "sum")
    assert float(loss) == pytest.approx(float(golden[f"ce_rand_{case}_loss"]), rel=1e-4)
    ok, err = rel_close(grad, golden[f"ce_rand_{case}_grad"], 1e-4)
    assert ok, err


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("reduction", ["mean", "sum", "none"])
@pytest.mark.parametrize("ls,cap,lss", [(0.0, None, 0.0), (0.1, None, 0.0), (0.0, 30.0, 0.0), (0.1, 5.0, 1e-4)])
def test_ce_liger_semantics(dtype, reduction, ls, cap, lss):
    rng = np.random.default_rng(0)
    rows, v = 64, 5003
    z = rng.normal(0, 3, (rows, v)).astype(np.float32)
    t = rng.integers(0, v, rows)
    t[rng.random(rows) < 0.1] = -100
    zin = torch.tensor(z, dtype=dtype).float().numpy()  # oracle on the rounded inputs
    ref_loss, ref_rows, _, ref_grad = liger_ref.ce(zin, t, ignore_index=-100, label_smoothing=ls, softcap=cap,
                                                   lse_square_scale=lss, reduction=reduction)
    loss, grad = run_ce(z, t, dtype, label_smoothing=ls, softcap=cap, lse_square_scale=lss, reduction=reduction)
    tol = TOL[dtype]
    ok, err = rel_close(loss, ref_loss, tol)
    assert ok, ("loss", err)
    ok, err = rel_close(grad, ref_grad, tol)
    assert ok, ("grad", err)
    # ignored rows: exactly zero gradient and loss
    assert np.all(grad[t == -100] == 0.0)
    if reduction == "none":
        assert np.all(loss[t == -100] == 0.0)


def test_ce_large_vocab_bf16_rows_sum_to_zero():
    rows, v = 256, 128256
    g = torch.Generator(device="cuda").manual_seed(1)
    x = (torch.randn(rows, v, device="cuda", generator=g) * 2).to(torch.bfloat16).requires_grad_(True)
    t = torch.randint(0, v, (rows,), device="cuda", generator=g)
    ref = torch.nn.functional.cross_entropy(x.detach().float(), t, reduction="sum")  # before: CE is in place
    loss = lk.LigerCrossEntropyLoss(reduction="sum")(x, t)
    loss.backward()
    assert loss.item() == pytest.approx(ref.item(), rel=2e-2)
    rs = x.grad.float().sum(dim=1)
    assert rs.abs().max().item() < 5e-2  # bf16 rounding of ~1e5 entries per row


@pytest.mark.parametrize("v,dtype", [(32000, torch.bfloat16), (128256, torch.bfloat16), (256000, torch.bfloat16),
                                     (128256, torch.float32), (40000, torch.float16), (5003, torch.bfloat16),
                                     (1000, torch.float32), (8192, torch.bfloat16)])
def test_ce_ring_path_matches_other_paths(v, dtype):
    """Default persistent TMA-ring kernel vs the one-CTA-per-row kernel, and the oracle."""
    rows = 300  # > SM count: several rows per persistent CTA
    g = torch.Generator(device="cuda").manual_seed(v)
    z = (torch.randn(rows, v, device="cuda", generator=g) * 3).to(dtype)
    t = torch.randint(0, v, (rows,), device="cuda", generator=g)
    t[::5] = -100
    t[1] = v - 1  # target in the ragged last piece
    kw = dict(label_smoothing=0.1, softcap=20.0, lse_square_scale=1e-4)

    def run():
        x = z.clone().requires_grad_(True)
        loss = lk.LigerCrossEntropyLoss(reduction="none", **kw)(x, t)
        loss.sum().backward()
        return loss.detach().float(), x.grad.float()

    l1, g1 = run()
    with _capi.select_path(_capi.PATH_CE_IMPL, 1):
        l2, g2 = run()
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    ok, err = rel_close(l1.cpu().numpy(), l2.cpu().numpy(), tol)
    assert ok, err
    ok, err = rel_close(g1.cpu().numpy(), g2.cpu().numpy(), tol)
    assert ok, err
    sel = [0, 1, 2, 3, 4, 5, 6, 7, 150, 299]
    _, rrows, _, rgrad = liger_ref.ce(z[sel].double().cpu().numpy(), t[sel].cpu().numpy(), reduction="none", **kw)
    ok, err = rel_close(l1[sel].cpu().numpy(), rrows, TOL.get(dtype, 2e-2))
    assert ok, err
    ok, err = rel_close(g1[sel].cpu().numpy(), rgrad, TOL.get(dtype, 2e-2))
    assert ok, err
    assert torch.all(g1[t == -100] == 0)
    assert torch.all(l1[t == -100] == 0)


def test_ce_ring_plain_mean_and_no_grad():
    """Ring kernel without options (no cap / smoothing), MEAN reduction, and the loss-only path."""
    rows, v = 777, 128256
    g = torch.Generator(device="cuda").manual_seed(1)
    z = torch.randn(rows, v, device="cuda", generator=g).to(torch.bfloat16)
    t = torch.randint(0, v, (rows,), device="cuda", generator=g)
    t[::7] = -100
    x = z.clone().requires_grad_(True)
    loss = lk.LigerCrossEntropyLoss()(x, t)
    loss.backward()
    ref = torch.nn.functional.cross_entropy(z.float(), t, ignore_index=-100)
    assert abs(loss.item() - ref.item()) <= 2e-3 * abs(ref.item())
    zr = z.float().requires_grad_(True)
    torch.nn.functional.cross_entropy(zr, t, ignore_index=-100).backward()
    ok, err = rel_close(x.grad.float().cpu().numpy(), zr.grad.cpu().numpy(), 2e-2)
    assert ok, err
    with torch.no_grad():
        l2 = lk.LigerCrossEntropyLoss()(z.clone(), t)
    assert abs(l2.item() - loss.item()) <= 1e-6 * abs(loss.item())


def test_ce_inplace_and_backward_scale():
    rows, v = 8, 100
    x = torch.randn(rows, v, device="cuda", requires_grad=True)
    t = torch.randint(0, v, (rows,), device="cuda")
    loss = lk.LigerCrossEntropyLoss()(x * 1.0, t)
    (3.0 * loss).backward()
    ref_x = x.detach().clone().requires_grad_(True)
    (3.0 * torch.nn.functional.cross_entropy(ref_x, t)).backward()
    torch.testing.assert_close(x.grad, ref_x.grad, rtol=1e-4, atol=1e-6)


def test_ce_target_out_of_range_raises():
    x = torch.randn(4, 10, device="cuda", requires_grad=True)
    t = torch.tensor([0, 1, 10, 2], device="cuda")
    with pytest.raises(errors.TargetOutOfRange):
        lk.LigerCrossEntropyLoss()(x, t)


def test_ce_mean_is_sum_over_count_exact_count():
    rows, v = 33, 77
    x = torch.randn(rows, v, device="cuda")
    t = torch.randint(0, v, (rows,), device="cuda")
    t[::3] = -100
    n = int((t != -100).sum())
    lm = lk.LigerCrossEntropyLoss(reduction="mean")(x.clone(), t)
    lsum = lk.LigerCrossEntropyLoss(reduction="sum")(x.clone(), t)
    assert lm.item() == pytest.approx(lsum.item() / n, rel=1e-6)


def test_rowfuse_inplace_contract_port_vs_gpu(golden):
    """The reference mutates logits into the gradient (rowfuse/ops.py:546-551); so do we."""
    x_np = golden["ce_rand_a_logits"]
    x = torch.tensor(x_np, dtype=torch.float32, device="cuda", requires_grad=True)
    t = torch.tensor(golden["ce_rand_a_target"], device="cuda")
    buf = x.detach()
    from paper_2410_10989_b200.cross_entropy import cross_entropy_forward

    loss, _, _, _, g = cross_entropy_forward(buf, t, compute_grad=True)
    assert g.data_ptr() == buf.data_ptr()
    ref = x_np.copy()
    rp.cross_entropy_(ref, golden["ce_rand_a_target"], mean=True)
    ok, err = rel_close(buf.cpu().numpy(), ref, 1e-4)
    assert ok, err


@pytest.mark.parametrize("impl", ["ring", "block"])
@pytest.mark.parametrize("reduction", ["mean", "sum", "none"])
@pytest.mark.parametrize("cap", [None, 20.0])
def test_ce_token_accuracy_and_predicted_tokens(impl, reduction, cap, path_knob):
    """Liger return_token_accuracy / return_predicted_tokens (LK/ops/cross_entropy.py:131-163, 294-299, 415-420)."""
    path_knob(_capi.PATH_CE_IMPL, {"ring": 0, "block": 1}[impl])
    rows, v = 300, 32000
    g = torch.Generator(device="cuda").manual_seed(7)
    z = (torch.randn(rows, v, device="cuda", generator=g) * 3).to(torch.bfloat16)
    t = torch.randint(0, v, (rows,), device="cuda", generator=g)
    zz = z.float() if cap is None else (cap * torch.tanh(z.float() / cap))
    t[::3] = zz[::3].argmax(1)  # a third of the rows predicted correctly
    t[::7] = -100
    x = z.clone().requires_grad_(True)
    out = lk.LigerCrossEntropyLoss(reduction=reduction, softcap=cap, return_token_accuracy=True,
                                   return_predicted_tokens=True)(x, t)
    want_pred = zz.argmax(1)
    want_pred[t == -100] = -1
    pred = out.predicted_tokens
    ign = t == -100
    if cap is None:
        assert torch.equal(pred, want_pred)
    else:  # bf16 tanh.approx vs torch tanh: a near-tie may resolve to a neighbour within one ulp
        assert (pred == want_pred).float().mean().item() > 0.99
        assert torch.all(pred[ign] == -1)
    correct = ((pred == t) & ~ign).float()
    if reduction == "none":
        assert torch.equal(out.token_accuracy, correct)
    else:
        assert abs(out.token_accuracy.item() - correct.sum().item() / (~ign).sum().item()) < 1e-6
    out.loss.sum().backward()  # gradients are unaffected by the options
    ref = lk.LigerCrossEntropyLoss(reduction=reduction, softcap=cap)
    x2 = z.clone().requires_grad_(True)
    ref(x2, t).sum().backward()
    assert torch.equal(x.grad, x2.grad)


def test_ce_int64_offsets_beyond_2_31_elements():
    """Logits with > 2^31 elements (8448 x 256000 bf16 = 4.3 GB, cfg4's vocabulary): rows past
    element 2^31 are addressed with 64-bit offsets; they match the oracle."""
    rows, v = 8448, 256000
    assert rows * v > 2**31
    g = torch.Generator(device="cuda").manual_seed(9)
    t = torch.randint(0, v, (rows,), device="cuda", generator=g)
    t[-3] = -100
    x = torch.empty(rows, v, dtype=torch.bfloat16, device="cuda")
    x.normal_(generator=g)
    sel = torch.tensor([0, rows // 2, rows - 4, rows - 3, rows - 2, rows - 1], device="cuda")
    ref_in = x[sel].double().cpu().numpy()
    x.requires_grad_(True)
    loss = lk.LigerCrossEntropyLoss(reduction="none")(x, t)
    loss.sum().backward()
    _, rrows, _, rgrad = liger_ref.ce(ref_in, t[sel].cpu().numpy(), reduction="none")
    ok, err = rel_close(loss.detach()[sel].float().cpu().numpy(), rrows, 2e-2)
    assert ok, err
    ok, err = rel_close(x.grad[sel].float().cpu().numpy(), rgrad, 2e-2)
    assert ok, err
    assert torch.all(x.grad[rows - 3] == 0) and loss[rows - 3].item() == 0.0


@pytest.mark.parametrize("impl", ["ring", "block"])
@pytest.mark.parametrize("reduction", ["mean", "sum", "none"])
@pytest.mark.parametrize("kw", [dict(), dict(softcap=20.0, lse_square_scale=1e-4), dict(label_smoothing=0.1),
                                dict(label_smoothing=0.2, softcap=20.0, lse_square_scale=1e-4)])
def test_ce_class_weights(impl, reduction, kw, path_knob):
    """Liger `weight` (class weights, LK/ops/cross_entropy.py:122-124, 165-171, 220-239, 278-288),
    with and without label smoothing, vs the float64 oracle (itself pinned to torch
    F.cross_entropy(weight=, label_smoothing=))."""
    path_knob(_capi.PATH_CE_IMPL, {"ring": 0, "block": 1}[impl])
    rows, v = 300, 4096
    g = torch.Generator(device="cuda").manual_seed(13)
    z = (torch.randn(rows, v, device="cuda", generator=g) * 3).to(torch.bfloat16)
    t = torch.randint(0, v, (rows,), device="cuda", generator=g)
    t[::6] = -100
    w = torch.rand(v, device="cuda", generator=g) + 0.1
    x = z.clone().requires_grad_(True)
    loss = lk.LigerCrossEntropyLoss(weight=w, reduction=reduction, **kw)(x, t)
    loss.sum().backward()
    rl, _, _, rg = liger_ref.ce(z.double().cpu().numpy(), t.cpu().numpy(), weight=w.double().cpu().numpy(),
                                reduction=reduction, **kw)
    ok, err = rel_close(loss.detach().float().cpu().numpy(), rl, 2e-2)
    assert ok, err
    ok, err = rel_close(x.grad.float().cpu().numpy(), rg, 2e-2)
    assert ok, err


def test_ce_unaligned_logits_vs_oracle():
    """Logits at a storage offset that breaks 16-byte alignment: the ring kernel declines, the
    block kernel's scalar path takes the rows."""
    rows, v = 64, 3001
    g = torch.Generator(device="cuda").manual_seed(17)
    base = (torch.randn(rows * v + 1, device="cuda", generator=g) * 3).to(torch.bfloat16)
    z = base[1:].view(rows, v)
    t = torch.randint(0, v, (rows,), device="cuda", generator=g)
    t[::5] = -100
    x = base.clone()[1:].view(rows, v).requires_grad_(True)
    loss = lk.LigerCrossEntropyLoss(label_smoothing=0.1)(x, t)
    loss.backward()
    rl, _, _, rg = liger_ref.ce(z.double().cpu().numpy(), t.cpu().numpy(), label_smoothing=0.1)
    assert rel_close(loss.item(), rl, 2e-2)[0]
    ok, err = rel_close(x.grad.float().cpu().numpy(), rg, 2e-2)
    assert ok, err


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("spread", [60.0, 1000.0])
def test_ce_extreme_logit_spread_stable(dtype, spread):
    """Online softmax with huge logit ranges (one dominant logit per row, the rest spread by
    `spread`): loss = lse - z_t exactly as Liger (no log(max(p, tiny)) clamp, SURVEY §8(a)
    edge-case note), gradients finite, against the float64 oracle.  Rows span the ring's
    multi-piece path (V = 40000)."""
    rng = np.random.default_rng(7)
    rows, v = 16, 40000
    z = rng.uniform(-spread, 0.0, (rows, v)).astype(np.float32)
    hot = rng.integers(0, v, rows)
    z[np.arange(rows), hot] = spread  # one dominant logit per row
    t = np.where(np.arange(rows) % 2 == 0, hot, rng.integers(0, v, rows))  # half hit it, half miss
    zin = torch.tensor(z, dtype=dtype).float().numpy()
    ref_loss, ref_rows, _, ref_grad = liger_ref.ce(zin, t, reduction="none")
    loss, grad = run_ce(z, t, dtype, reduction="none")
    assert np.all(np.isfinite(loss)) and np.all(np.isfinite(grad))
    assert rel_close(loss, ref_rows, TOL[dtype])[0]
    assert rel_close(grad, ref_grad, TOL[dtype])[0]
