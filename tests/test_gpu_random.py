"""Seeded random configurations of the row ops and the standalone cross entropy against the
float64 oracle (GPU).

Each op gets 16 configurations over its shape edges: ragged widths (not multiples of the
16-byte vector), widths past the register kernels, single rows, and every dtype. The
options are drawn too (RMSNorm offset, label smoothing, softcap, z-loss, reductions,
ignored targets). The tolerance is the north-star one for the dtype: 1e-4 in fp32,
2e-2 in bf16 / fp16. The oracle is evaluated on the dtype-rounded inputs.
"""

import math

import numpy as np
import pytest
import torch

import paper_2410_10989_b200 as lk
from oracle import liger_ref
from oracle import rowfuse_port as rp
from tests.conftest import rel_close

pytestmark = pytest.mark.gpu

DTYPES = [torch.float32, torch.bfloat16, torch.float16]
TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2, torch.float16: 2e-2}


def _cases(seed, n=16):
    rng = np.random.default_rng(seed)
    return [(i, DTYPES[i % 3], int(rng.choice([1, 3, 64, 257, 1000])), int(rng.choice([8, 24, 100, 512, 1000, 4096,
                                                                                       5000])),
             int(rng.integers(0, 1 << 30))) for i in range(n)]


def _t(a, dtype):
    return torch.tensor(a, dtype=dtype, device="cuda")


def _r(t):  # dtype-rounded float64 copy on the host
    return t.detach().double().cpu().numpy()


@pytest.mark.parametrize("case", _cases(11), ids=lambda c: f"c{c[0]}")
def test_rmsnorm_random_vs_oracle(case):
    i, dtype, rows, cols, seed = case
    rng = np.random.default_rng(seed)
    offset = float(rng.choice([0.0, 1.0]))
    x = _t(rng.uniform(-2, 2, (rows, cols)), dtype).requires_grad_(True)
    w = _t(rng.uniform(0.5, 1.5, cols), dtype).requires_grad_(True)
    dy = _t(rng.uniform(-1, 1, (rows, cols)), dtype)
    # casting 'gemma' computes in fp32 throughout: the mode the float64 oracle restates
    y = lk.LigerRMSNormFunction.apply(x, w, 1e-6, offset, "gemma", False)
    y.backward(dy)
    ry, _ = liger_ref.rmsnorm_fwd(_r(x), _r(w), 1e-6, offset)
    rdx, rdw = liger_ref.rmsnorm_bwd(_r(dy), _r(x), _r(w), 1e-6, offset)
    tol = TOL[dtype]
    assert rel_close(_r(y), ry, tol)[0]
    assert rel_close(_r(x.grad), rdx, tol)[0]
    assert rel_close(_r(w.grad), rdw, tol)[0]


@pytest.mark.parametrize("case", _cases(12), ids=lambda c: f"c{c[0]}")
def test_layernorm_random_vs_oracle(case):
    i, dtype, rows, cols, seed = case
    rng = np.random.default_rng(seed)
    x = _t(rng.uniform(-2, 2, (rows, cols)) + rng.normal() * 3, dtype).requires_grad_(True)
    w = _t(rng.uniform(0.5, 1.5, cols), dtype).requires_grad_(True)
    b = _t(rng.normal(size=cols), dtype).requires_grad_(True)
    dy = _t(rng.uniform(-1, 1, (rows, cols)), dtype)
    y = lk.liger_layer_norm(x, w, b, 1e-6)
    y.backward(dy)
    ry, mu, r = rp.layernorm_forward(_r(x), _r(w), _r(b), 1e-6)
    rdx, rdw, rdb = rp.layernorm_backward(_r(dy), _r(x), mu, r, _r(w))
    tol = TOL[dtype]
    assert rel_close(_r(y), ry, tol)[0]
    assert rel_close(_r(x.grad), rdx, tol)[0]
    assert rel_close(_r(w.grad), rdw, tol)[0]
    assert rel_close(_r(b.grad), rdb, tol)[0]


@pytest.mark.parametrize("case", _cases(13), ids=lambda c: f"c{c[0]}")
def test_glu_random_vs_oracle(case):
    i, dtype, rows, cols, seed = case
    rng = np.random.default_rng(seed)
    gelu = bool(i % 2)
    a = _t(rng.uniform(-4, 4, (rows, cols)), dtype).requires_grad_(True)
    b = _t(rng.uniform(-2, 2, (rows, cols)), dtype).requires_grad_(True)
    dc = _t(rng.uniform(-1, 1, (rows, cols)), dtype)
    fn = lk.LigerGELUMulFunction if gelu else lk.LigerSiLUMulFunction
    ra, rb, rdc = _r(a), _r(b), _r(dc)
    c = fn.apply(a, b)
    c.backward(dc)
    fwd, bwd = (rp.geglu_forward, rp.geglu_backward) if gelu else (rp.swiglu_forward, rp.swiglu_backward)
    rda, rdb = bwd(rdc, ra, rb)
    tol = TOL[dtype]
    assert rel_close(_r(c), fwd(ra, rb), tol)[0]
    assert rel_close(_r(a.grad), rda, tol)[0]
    assert rel_close(_r(b.grad), rdb, tol)[0]


@pytest.mark.parametrize("case", _cases(14), ids=lambda c: f"c{c[0]}")
def test_rope_random_vs_oracle(case):
    i, dtype, _, _, seed = case
    rng = np.random.default_rng(seed)
    bsz, seq = int(rng.choice([1, 2, 3])), int(rng.choice([1, 5, 64, 130]))
    nq, nk = [(1, 1), (4, 1), (8, 2), (32, 8), (6, 3)][i % 5]
    d = int(rng.choice([8, 16, 64, 128]))
    per_batch = bool(rng.random() < 0.3)
    cos, sin = liger_ref.rope_tables(seq, d, 500000.0, batch=bsz if per_batch else 1)
    q = _t(rng.normal(size=(bsz, nq, seq, d)), dtype)
    k = _t(rng.normal(size=(bsz, nk, seq, d)), dtype)
    cs, sn = _t(cos, dtype), _t(sin, dtype)
    # the oracle first: the op rotates in place, and with one head `.contiguous()` of the
    # transposed view is the same storage as `k`
    rq, rk = liger_ref.rope(_r(q), _r(k), _r(cs), _r(sn))
    # the HF layout: (B, n_heads, T, d) views of (B, T, n_heads, d) storage
    qv = q.clone().transpose(1, 2).contiguous().transpose(1, 2).requires_grad_(True)
    kv = k.clone().transpose(1, 2).contiguous().transpose(1, 2).requires_grad_(True)
    qo, ko = lk.liger_rotary_pos_emb(qv, kv, cs, sn)
    dq = _t(rng.normal(size=qo.shape), dtype)
    dk = _t(rng.normal(size=ko.shape), dtype)
    gq, gk = liger_ref.rope(_r(dq), _r(dk), _r(cs), _r(sn), backward=True)  # before: grads rotate in place too
    torch.autograd.backward([qo, ko], [dq, dk])
    tol = TOL[dtype]
    assert rel_close(_r(qo), rq, tol)[0] and rel_close(_r(ko), rk, tol)[0]
    assert rel_close(_r(qv.grad), gq, tol)[0] and rel_close(_r(kv.grad), gk, tol)[0]


@pytest.mark.parametrize("case", _cases(15), ids=lambda c: f"c{c[0]}")
def test_cross_entropy_random_vs_oracle(case):
    i, dtype, rows, _, seed = case
    rng = np.random.default_rng(seed)
    v = int(rng.choice([2, 37, 1000, 8229, 40000]))
    opts = dict(reduction=str(rng.choice(["mean", "sum", "none"])))
    if rng.random() < 0.4:
        opts["label_smoothing"] = float(rng.choice([0.05, 0.2]))
    if rng.random() < 0.3:
        opts["softcap"] = float(rng.choice([3.0, 30.0]))
    if rng.random() < 0.2:
        opts["lse_square_scale"] = 1e-3
    z = _t(rng.normal(0, 3, (rows, v)), dtype)
    t = rng.integers(0, v, rows)
    t[rng.random(rows) < 0.2] = -100
    ref_loss, ref_rows, _, ref_grad = liger_ref.ce(_r(z), t, **opts)
    zz = z.clone().requires_grad_(True)
    loss = lk.LigerCrossEntropyLoss(**opts)(zz, torch.tensor(t, device="cuda"))
    (loss.sum() if opts["reduction"] == "none" else loss).backward()
    tol = TOL[dtype]
    if opts["reduction"] == "none":
        assert rel_close(_r(loss.detach()), ref_rows, tol)[0]
    else:
        assert loss.item() == pytest.approx(ref_loss, rel=tol, abs=tol * 1e-3)
    assert rel_close(_r(zz.grad), ref_grad, tol)[0]
    assert torch.all(zz.grad[torch.tensor(t == -100, device="cuda")] == 0)
    assert math.isfinite(float(_r(loss.detach()).sum()))
