"""Ignored-row skipping around the FLCE (csrc/compact.cu, fused_linear_cross_entropy.py
`_forward_kept_rows`) (GPU).

The compaction map is checked bit for bit against numpy, the row gather for every element
width and fill, and the FLCE with skipping on against the float64 oracle and against the same
call with skipping off, over the Liger options.  Rows whose target is ignore_index must come
back exactly as the full call leaves them: loss 0, gradient row 0, predicted token -1.
"""

import numpy as np
import pytest
import torch

import paper_2410_10989_b200.fused_linear_cross_entropy as flce_mod
from oracle import liger_ref
from paper_2410_10989_b200 import _capi
from tests.conftest import rel_close

pytestmark = pytest.mark.gpu


def _st():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("rows,frac,ign", [(0, 0.1, -100), (1, 1.0, -100), (1, 0.0, -100), (1000, 0.1, -100),
                                           (8192, 0.1, -100), (8192, 0.0, -100), (8192, 1.0, -100),
                                           (70001, 0.35, -100), (5000, 0.5, 7)])
def test_compact_rows_matches_numpy(rows, frac, ign):
    rng = np.random.default_rng(rows + int(frac * 100))
    t = rng.integers(0, 50, rows)
    t[rng.random(rows) < frac] = ign
    td = torch.tensor(t, dtype=torch.int64, device="cuda")
    index = torch.full((max(rows, 1),), 123, dtype=torch.int64, device="cuda")
    pos = torch.full((max(rows, 1),), 123, dtype=torch.int64, device="cuda")
    count = torch.empty(1, dtype=torch.int64, device="cuda")
    L = _capi.load()
    assert L.lk_compact_rows(td.data_ptr(), rows, ign, index.data_ptr(), pos.data_ptr(), count.data_ptr(), _st()) == 0
    keep = np.nonzero(t != ign)[0]
    want_pos = np.full(rows, -1)
    want_pos[keep] = np.arange(len(keep))
    assert int(count.item()) == len(keep)
    got_index = index.cpu().numpy()[:rows]
    assert np.array_equal(got_index[:len(keep)], keep)
    assert np.all(got_index[len(keep):] == -1)
    assert np.array_equal(pos.cpu().numpy()[:rows], want_pos)


@pytest.mark.parametrize("dtype,cols", [(torch.bfloat16, 4096), (torch.bfloat16, 100), (torch.float32, 1),
                                        (torch.int64, 1), (torch.uint8, 3), (torch.float32, 96),
                                        (torch.float16, 1000)])
def test_gather_rows_every_width_and_fill(dtype, cols):
    rng = np.random.default_rng(cols)
    rows_src, rows_out = 300, 517
    src = torch.tensor(rng.integers(0, 100, (rows_src, cols)), device="cuda").to(dtype)
    idx = rng.integers(-1, rows_src, rows_out)
    dst = torch.empty(rows_out, cols, dtype=dtype, device="cuda")
    fill = torch.tensor([-1 if dtype == torch.int64 else 0], dtype=dtype)
    fill_bits = int.from_bytes(fill.numpy().tobytes() if dtype != torch.bfloat16 else fill.view(torch.int16).numpy().tobytes(),
                               "little")
    L = _capi.load()
    idx_d = torch.tensor(idx, dtype=torch.int64, device="cuda")
    assert L.lk_gather_rows(src.data_ptr(), cols, src.element_size(), idx_d.data_ptr(), rows_out, dst.data_ptr(),
                            fill_bits, _st()) == 0
    want = src.cpu()[torch.tensor(np.maximum(idx, 0))]
    want[torch.tensor(idx < 0)] = fill.to(dtype)
    assert torch.equal(dst.cpu(), want)


def _problem(bt, h, v, frac, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.rand(bt, h, device="cuda", generator=g) * 2 - 1).to(dtype)
    w = ((torch.rand(v, h, device="cuda", generator=g) * 2 - 1) / (h ** 0.5) * 3).to(dtype)
    t = torch.randint(0, v, (bt,), device="cuda", generator=g)
    t[torch.rand(bt, device="cuda", generator=g) < frac] = -100
    return x, w, t


CASES = [dict(), dict(reduction="sum"), dict(reduction="none"), dict(lse_square_scale=1e-4, return_z_loss=True),
         dict(lse_square_scale=1e-4, return_z_loss=True, reduction="none"),
         dict(label_smoothing=0.1, softcap=30.0), dict(return_token_accuracy=True, return_predicted_tokens=True),
         dict(return_token_accuracy=True, return_predicted_tokens=True, reduction="none"),
         dict(_ce_weight=True), dict(_ce_weight=True, label_smoothing=0.1), dict(_bias=True),
         dict(accum_dtype=torch.float32), dict(use_token_scaling=True), dict(_dtype=torch.float32),
         dict(_frac=0.9), dict(_frac=1.0), dict(_frac=0.0), dict(_dtype=torch.float16),
         dict(_no_grad_x=True), dict(_no_grad_x=True, _bias=True)]


@pytest.mark.parametrize("device_count", [False, True], ids=["host_count", "device_count"])
@pytest.mark.parametrize("kw", CASES, ids=lambda k: "-".join(f"{a}" for a in k) or "default")
def test_flce_skip_ignored_rows_vs_full_call_and_oracle(kw, device_count, monkeypatch):
    """device_count: the kept-row count stays on the device (KEPT_ROWS_DEVICE_COUNT, the CUDA
    graph path): all row slots run, and the CTA-pair GEMMs skip the work past the count."""
    monkeypatch.setattr(flce_mod, "COMPACT_MIN_SKIPPED", 1)
    monkeypatch.setattr(flce_mod, "KEPT_ROWS_DEVICE_COUNT", device_count)
    kw = dict(kw)
    dtype = kw.pop("_dtype", torch.bfloat16)
    frac = kw.pop("_frac", 0.3)
    bt, h, v = 700, 256, 3000
    x, w, t = _problem(bt, h, v, frac, dtype, seed=len(str(kw)))
    if kw.pop("_ce_weight", False):
        kw["ce_weight"] = torch.rand(v, device="cuda") + 0.2
    if kw.pop("_bias", False):
        kw["bias"] = (torch.rand(v, device="cuda") * 0.2).to(dtype)
    need_gx = not kw.pop("_no_grad_x", False)
    common = dict(compute_grad_input=need_gx, compute_grad_weight=True, chunk_rows=256, **kw)
    on = flce_mod.fused_linear_cross_entropy_forward(x, w, t, skip_ignored_rows=True, **common)
    off = flce_mod.fused_linear_cross_entropy_forward(x, w, t, skip_ignored_rows=False, **common)
    torch.cuda.synchronize()
    ign = t == -100
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    names = ["loss", "z_loss", "acc", "pred", "grad_x", "grad_w", "grad_b"]
    for name, a, b in zip(names, on, off):
        assert (a is None) == (b is None), name
        if a is None:
            continue
        assert a.shape == b.shape and a.dtype == b.dtype, name
        if name == "pred":
            assert torch.all(a[ign] == -1)
            assert (a == b).float().mean().item() > 0.99
            continue
        if name == "grad_x" or (a.dim() == 1 and a.numel() == bt):  # per-row outputs: ignored rows exact
            assert torch.all(a[ign] == 0), name
        assert rel_close(a.double().cpu().numpy(), b.double().cpu().numpy(), tol)[0], name
    # and against the float64 oracle
    ref_kw = {k: kw[k] for k in ("reduction", "label_smoothing", "lse_square_scale", "softcap") if k in kw}
    if "ce_weight" in kw:
        ref_kw["weight"] = kw["ce_weight"].double().cpu().numpy()
    if kw.get("use_token_scaling"):
        ref_kw["token_scaling"] = True
    b = kw.get("bias")
    rl, rrows, _, rgx, rgw, rgb = liger_ref.flce(x.double().cpu().numpy(), w.double().cpu().numpy(), t.cpu().numpy(),
                                                 bias=None if b is None else b.double().cpu().numpy(), **ref_kw)
    loss = on[0]
    if kw.get("reduction") == "none":
        assert rel_close(loss.double().cpu().numpy(), rrows, tol)[0]
    else:
        assert rel_close(float(loss.item()), rl, tol)[0]
    if need_gx:
        assert rel_close(on[4].double().cpu().numpy(), rgx, tol)[0]
    else:
        assert on[4] is None
    assert rel_close(on[5].double().cpu().numpy(), rgw, tol)[0]
    if b is not None and need_gx:
        assert rel_close(on[6].double().cpu().numpy(), rgb, tol)[0]


def test_skip_ignored_rows_is_bitwise_repeatable():
    x, w, t = _problem(8192, 512, 8192, 0.1, torch.bfloat16, seed=3)
    a = flce_mod.fused_linear_cross_entropy_forward(x, w, t, compute_grad_input=True, compute_grad_weight=True)
    for _ in range(3):
        b = flce_mod.fused_linear_cross_entropy_forward(x, w, t, compute_grad_input=True, compute_grad_weight=True)
        assert a[0].item() == b[0].item() and torch.equal(a[4], b[4]) and torch.equal(a[5], b[5])


@pytest.mark.parametrize("device_count", [True, False], ids=["device_count", "host_count"])
def test_prepared_kept_rows_match_and_are_consumed(device_count, monkeypatch):
    """lk.prepare_kept_rows on a side stream ahead of the call: the same result bit for bit as
    the call that compacts by itself; the entry is consumed; an in-place change to the targets
    after preparing (a new tensor version) falls back to a fresh compaction."""
    import paper_2410_10989_b200 as lk

    monkeypatch.setattr(flce_mod, "KEPT_ROWS_DEVICE_COUNT", device_count)
    flce_mod._PREPARED.clear()
    x, w, t = _problem(4096, 256, 5000, 0.25, torch.bfloat16, seed=9)
    kw = dict(compute_grad_input=True, compute_grad_weight=True)
    ref = flce_mod.fused_linear_cross_entropy_forward(x, w, t, **kw)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    kr = lk.prepare_kept_rows(t, stream=side)
    assert kr is not None and len(flce_mod._PREPARED) == 1
    torch.cuda.current_stream().wait_stream(side)
    got = flce_mod.fused_linear_cross_entropy_forward(x, w, t, **kw)
    assert len(flce_mod._PREPARED) == 0
    assert ref[0].item() == got[0].item() and torch.equal(ref[4], got[4]) and torch.equal(ref[5], got[5])
    assert kr.n == int((t != -100).sum())
    # stale: the targets change after preparing -> recompacted, matches a fresh call
    lk.prepare_kept_rows(t)
    t2 = t.clone()
    t[:100] = -100
    t2[:100] = -100
    a = flce_mod.fused_linear_cross_entropy_forward(x, w, t, **kw)
    b = flce_mod.fused_linear_cross_entropy_forward(x, w, t2, **kw)
    assert a[0].item() == b[0].item() and torch.equal(a[4], b[4]) and torch.equal(a[5], b[5])
    flce_mod._PREPARED.clear()


@pytest.mark.parametrize("shape", [(8192, 512, 8192, 0.1), (3000, 256, 5000, 0.6), (700, 256, 3000, 1.0)])
def test_device_count_matches_host_count(shape, monkeypatch):
    """The device-count kept-row FLCE against the host-count one: loss and gradients within the
    bf16 tolerance (chunk grouping differs), ignored rows exact, bitwise repeatable."""
    bt, h, v, frac = shape
    x, w, t = _problem(bt, h, v, frac, torch.bfloat16, seed=bt)
    kw = dict(compute_grad_input=True, compute_grad_weight=True, chunk_rows=1024)
    monkeypatch.setattr(flce_mod, "COMPACT_MIN_SKIPPED", 1)
    monkeypatch.setattr(flce_mod, "KEPT_ROWS_DEVICE_COUNT", False)
    host = flce_mod.fused_linear_cross_entropy_forward(x, w, t, **kw)
    monkeypatch.setattr(flce_mod, "KEPT_ROWS_DEVICE_COUNT", True)
    dev = flce_mod.fused_linear_cross_entropy_forward(x, w, t, **kw)
    dev2 = flce_mod.fused_linear_cross_entropy_forward(x, w, t, **kw)
    assert dev[0].item() == dev2[0].item() and torch.equal(dev[4], dev2[4]) and torch.equal(dev[5], dev2[5])
    ign = t == -100
    assert torch.all(dev[4][ign] == 0)
    for a, b in ((dev[0], host[0]), (dev[4], host[4]), (dev[5], host[5])):
        assert rel_close(a.double().cpu().numpy(), b.double().cpu().numpy(), 2e-2)[0]


@pytest.mark.parametrize("case", ["cta1", "fp32_accumulator_fold", "grad_w_slices", "bias"])
def test_device_count_special_paths_vs_oracle(case, path_knob, monkeypatch):
    """Device-count kept rows where the unread-row shortcuts must stay off or stay safe: the
    single-CTA GEMM (ignores limits), a last chunk that folds the fp32 dW accumulator (reads every
    row), grad_w in vocab-row slices with events, and a bias gradient (column sum over all rows)."""
    monkeypatch.setattr(flce_mod, "KEPT_ROWS_DEVICE_COUNT", True)
    monkeypatch.setattr(flce_mod, "COMPACT_MIN_SKIPPED", 1)
    bt, h, v = 3000, 256, 4000
    x, w, t = _problem(bt, h, v, 0.35, torch.bfloat16, seed=77)
    kw = dict(compute_grad_input=True, compute_grad_weight=True, chunk_rows=1024)
    b = None
    if case == "cta1":
        path_knob(_capi.PATH_CTA_GROUP, 1)
    elif case == "fp32_accumulator_fold":
        kw["chunk_rows"] = 256  # 12 chunks > 8: fp32 accumulator, last chunk folds it into grad_w
    elif case == "grad_w_slices":
        kw["grad_w_slice_events"] = [torch.cuda.Event() for _ in range(4)]
    else:
        b = (torch.rand(v, device="cuda") * 0.2).to(torch.bfloat16)
        kw["bias"] = b
    out = flce_mod.fused_linear_cross_entropy_forward(x, w, t, **kw)
    torch.cuda.synchronize()
    rl, _, _, rgx, rgw, rgb = liger_ref.flce(x.double().cpu().numpy(), w.double().cpu().numpy(), t.cpu().numpy(),
                                             bias=None if b is None else b.double().cpu().numpy())
    assert rel_close(float(out[0].item()), rl, 2e-2)[0]
    assert rel_close(out[4].double().cpu().numpy(), rgx, 2e-2)[0]
    assert rel_close(out[5].double().cpu().numpy(), rgw, 2e-2)[0]
    assert torch.all(out[4][t == -100] == 0)
    assert torch.isfinite(out[5]).all()
    if b is not None:
        assert rel_close(out[6].double().cpu().numpy(), rgb, 2e-2)[0]
