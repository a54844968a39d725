"""RMSNorm, RoPE, SwiGLU/GeGLU on the GPU against the reference goldens and oracle (GPU)."""

import numpy as np
import pytest
import torch

import paper_2410_10989_b200 as lk
from paper_2410_10989_b200 import _capi
from oracle import liger_ref, rowfuse_port as rp
from tests.conftest import rel_close
from tests.torch_ref import close

pytestmark = pytest.mark.gpu


def cuda(a, dtype=torch.float32):
    return torch.tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


# ------------------------------------------------------------------ RMSNorm
def test_rmsnorm_fp32_vs_reference_golden(golden):
    x = cuda(golden["rms_x"]).requires_grad_(True)
    m = lk.LigerRMSNorm(33, eps=1e-6, casting_mode="gemma", in_place=False).cuda()
    with torch.no_grad():
        m.weight.copy_(cuda(golden["rms_gamma"]))
    y = m(x)
    y.backward(cuda(golden["rms_dy"]))
    assert rel_close(y.detach().cpu().numpy(), golden["rms_y"], 1e-4)[0]
    assert rel_close(x.grad.cpu().numpy(), golden["rms_dx"], 1e-4)[0]
    assert rel_close(m.weight.grad.cpu().numpy(), golden["rms_dgamma"], 1e-4)[0]


@pytest.mark.parametrize("mode", ["llama", "gemma", "none"])
@pytest.mark.parametrize("shape", [(8192, 4096), (37, 1000), (5, 4099)])
def test_rmsnorm_bf16_vs_oracle(mode, shape):
    rows, cols = shape
    g = torch.Generator(device="cuda").manual_seed(rows + cols)
    x = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = (torch.rand(cols, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
    dy = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    offset = 0.0 if mode != "gemma" else 1.0
    xr = x.clone().requires_grad_(True)
    wr = w.clone().requires_grad_(True)
    y = lk.liger_rms_norm(xr, wr, 1e-6, offset, mode, False)
    y.backward(dy)
    sel = slice(0, min(rows, 512))
    ry, _ = liger_ref.rmsnorm_fwd(x[sel].double().cpu().numpy(), w.double().cpu().numpy(), 1e-6, offset)
    rdx, _ = liger_ref.rmsnorm_bwd(dy[sel].double().cpu().numpy(), x[sel].double().cpu().numpy(),
                                   w.double().cpu().numpy(), 1e-6, offset)
    ok, err = rel_close(y[sel].float().detach().cpu().numpy(), ry, 2e-2)
    assert ok, ("y", err)
    ok, err = rel_close(xr.grad[sel].float().cpu().numpy(), rdx, 2e-2)
    assert ok, ("dx", err)
    # dW over all rows against a torch fp32 restatement
    xf, dyf = x.float(), dy.float()
    r = torch.rsqrt((xf * xf).mean(1, keepdim=True) + 1e-6)
    rdw = (dyf * xf * r).sum(0)
    assert close(wr.grad, rdw, 2e-2)


@pytest.mark.parametrize("impl", ["ring", "warp", "generic"])
@pytest.mark.parametrize("shape,dtype", [((8192, 4096), torch.bfloat16), ((300, 1000), torch.bfloat16),
                                         ((37, 1000), torch.bfloat16), ((1000, 2048), torch.float32),
                                         ((513, 256), torch.float16), ((3, 64), torch.bfloat16)])
@pytest.mark.parametrize("mode", ["llama", "gemma", "none"])
def test_rmsnorm_default_matches_other_paths(impl, shape, dtype, mode):
    """Default (CTA register) kernels vs the TMA-ring, register-warp and generic kernels."""
    rows, cols = shape
    g = torch.Generator(device="cuda").manual_seed(rows * 7 + cols)
    x = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(dtype)
    w = (torch.rand(cols, device="cuda", generator=g) + 0.5).to(dtype)
    dy = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(dtype)
    offset = 1.0 if mode == "gemma" else 0.0

    def run(in_place):
        xr = x.clone().requires_grad_(True)
        wr = w.clone().requires_grad_(True)
        y = lk.liger_rms_norm(xr, wr, 1e-6, offset, mode, in_place)
        y.backward(dy.clone())
        return y.detach().float(), xr.grad.float(), wr.grad.float()

    a = run(True)
    with _capi.select_path(_capi.PATH_NORM_IMPL, {"warp": 1, "generic": 2, "ring": 3}[impl]):
        b = run(False)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    for name, u, v in zip(("y", "dx", "dw"), a, b):
        ok, err = rel_close(u.cpu().numpy(), v.cpu().numpy(), tol)
        assert ok, (name, err)
    sel = slice(0, min(rows, 256))
    ry, _ = liger_ref.rmsnorm_fwd(x[sel].double().cpu().numpy(), w.double().cpu().numpy(), 1e-6, offset)
    rdx, _ = liger_ref.rmsnorm_bwd(dy[sel].double().cpu().numpy(), x[sel].double().cpu().numpy(),
                                   w.double().cpu().numpy(), 1e-6, offset)
    rt = 1e-4 if dtype == torch.float32 else 2e-2
    ok, err = rel_close(a[0][sel].cpu().numpy(), ry, rt)
    assert ok, ("y vs oracle", err)
    ok, err = rel_close(a[1][sel].cpu().numpy(), rdx, rt)
    assert ok, ("dx vs oracle", err)


def test_rmsnorm_dw_deterministic_and_batch_linear():
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(4096, 1024, device="cuda", generator=g)
    w = torch.randn(1024, device="cuda", generator=g)
    dy = torch.randn(4096, 1024, device="cuda", generator=g)
    outs = []
    for _ in range(2):
        wr = w.clone().requires_grad_(True)
        lk.liger_rms_norm(x, wr, 1e-6, 0.0, "gemma", False).backward(dy)
        outs.append(wr.grad.clone())
    assert torch.equal(outs[0], outs[1])  # fixed-order two-stage reduction


# ---------------------------------------------------------------- LayerNorm
def test_layernorm_fp32_vs_reference_golden(golden):
    x = cuda(golden["ln_x"]).requires_grad_(True)
    m = lk.LigerLayerNorm(40, eps=1e-6, bias=True).cuda()
    with torch.no_grad():
        m.weight.copy_(cuda(golden["ln_gamma"]))
        m.bias.copy_(cuda(golden["ln_beta"]))
    y = m(x)
    y.backward(cuda(golden["ln_dy"]))
    for name, a, b in (("y", y.detach(), golden["ln_y"]), ("dx", x.grad, golden["ln_dx"]),
                       ("dgamma", m.weight.grad, golden["ln_dgamma"]), ("dbeta", m.bias.grad, golden["ln_dbeta"])):
        ok, err = rel_close(a.cpu().numpy(), b, 1e-4)
        assert ok, (name, err)


@pytest.mark.parametrize("shape,dtype", [((8192, 4096), torch.bfloat16), ((300, 1000), torch.bfloat16),
                                         ((37, 2048), torch.float32), ((5, 64), torch.float16)])
def test_layernorm_vs_oracle_and_torch(shape, dtype):
    rows, cols = shape
    g = torch.Generator(device="cuda").manual_seed(rows + 3 * cols)
    x = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 0.7).to(dtype)
    w = (torch.rand(cols, device="cuda", generator=g) + 0.5).to(dtype)
    b = (torch.rand(cols, device="cuda", generator=g) - 0.5).to(dtype)
    dy = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(dtype)
    xr, wr, br = x.clone().requires_grad_(True), w.clone().requires_grad_(True), b.clone().requires_grad_(True)
    y = lk.liger_layer_norm(xr, wr, br, 1e-6)
    y.backward(dy)
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    sel = slice(0, min(rows, 256))
    xs = x[sel].double().cpu().numpy()
    ry, mu, r = rp.layernorm_forward(xs, w.double().cpu().numpy(), b.double().cpu().numpy())
    rdx, _, _ = rp.layernorm_backward(dy[sel].double().cpu().numpy(), xs, mu, r, w.double().cpu().numpy())
    ok, err = rel_close(y[sel].detach().float().cpu().numpy(), ry, tol)
    assert ok, ("y", err)
    ok, err = rel_close(xr.grad[sel].float().cpu().numpy(), rdx, tol)
    assert ok, ("dx", err)
    # dgamma / dbeta over all rows against torch fp32 autograd
    xf = x.float().requires_grad_(True)
    wf, bf = w.float().requires_grad_(True), b.float().requires_grad_(True)
    torch.nn.functional.layer_norm(xf, (cols,), wf, bf, eps=1e-6).backward(dy.float())
    assert close(wr.grad, wf.grad, tol) and close(br.grad, bf.grad, tol)


def test_layernorm_grads_deterministic():
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(4096, 1024, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(1024, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(1024, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(4096, 1024, device="cuda", generator=g).to(torch.bfloat16)
    outs = []
    for _ in range(2):
        xr, wr, br = x.clone().requires_grad_(True), w.clone().requires_grad_(True), b.clone().requires_grad_(True)
        lk.liger_layer_norm(xr, wr, br, 1e-6).backward(dy)
        outs.append((xr.grad.clone(), wr.grad.clone(), br.grad.clone()))
    assert all(torch.equal(p, q) for p, q in zip(*outs))


# --------------------------------------------------------------------- RoPE
def test_rope_fp32_vs_reference_golden(golden):
    q, k, th, pos = golden["rope_q"], golden["rope_k"], golden["rope_thetas"], golden["rope_pos"]
    rows, d = q.shape
    # golden rows are independent tokens: map to (B=1, T=rows, nh=1, d) with per-token tables
    ang = pos[:, None] * th[None, :]
    emb = np.concatenate([ang, ang], axis=-1)
    cos, sin = cuda(np.cos(emb)[None]), cuda(np.sin(emb)[None])
    qt = cuda(q).reshape(1, rows, 1, d).transpose(1, 2)
    kt = cuda(k).reshape(1, rows, 1, d).transpose(1, 2)
    qo, ko = lk.liger_rotary_pos_emb(qt, kt, cos, sin)
    assert rel_close(qo.transpose(1, 2).reshape(rows, d).cpu().numpy(), golden["rope_q_fwd"], 1e-4)[0]
    assert rel_close(ko.transpose(1, 2).reshape(rows, d).cpu().numpy(), golden["rope_k_fwd"], 1e-4)[0]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_rope_llama3_gqa_fwd_bwd(dtype):
    b, t, nq, nk, d = 4, 2048, 32, 8, 128
    g = torch.Generator(device="cuda").manual_seed(1)
    q0 = torch.randn(b, t, nq, d, device="cuda", generator=g).to(dtype)
    k0 = torch.randn(b, t, nk, d, device="cuda", generator=g).to(dtype)
    cos_np, sin_np = liger_ref.rope_tables(t, d, base=500000.0)
    cos, sin = cuda(cos_np, dtype), cuda(sin_np, dtype)
    q = q0.clone().transpose(1, 2).requires_grad_(True)
    k = k0.clone().transpose(1, 2).requires_grad_(True)
    qo, ko = lk.liger_rotary_pos_emb(q, k, cos, sin)
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    rq, rk = liger_ref.rope(q0[:1, :64].transpose(1, 2).double().cpu().numpy(),
                            k0[:1, :64].transpose(1, 2).double().cpu().numpy(),
                            cos.double().cpu().numpy()[:, :64], sin.double().cpu().numpy()[:, :64])
    assert rel_close(qo[:1, :, :64].float().detach().cpu().numpy(), rq, tol)[0]
    assert rel_close(ko[:1, :, :64].float().detach().cpu().numpy(), rk, tol)[0]
    # backward is the inverse rotation: grad of sum(qo * u) wrt q = R^T u
    u = torch.randn_like(qo)
    v = torch.randn_like(ko)
    u0, v0 = u.clone(), v.clone()  # the backward rotates the incoming gradients in place (Liger contract)
    torch.autograd.backward([qo, ko], [u, v])
    u, v = u0, v0
    bq, bk = liger_ref.rope(u[:1, :, :64].double().cpu().numpy(), v[:1, :, :64].double().cpu().numpy(),
                            cos.double().cpu().numpy()[:, :64], sin.double().cpu().numpy()[:, :64], backward=True)
    assert rel_close(q.grad[:1, :, :64].float().cpu().numpy(), bq, tol)[0]
    assert rel_close(k.grad[:1, :, :64].float().cpu().numpy(), bk, tol)[0]


def test_rope_per_batch_tables():
    b, t, nq, nk, d = 2, 16, 4, 2, 64
    q0 = torch.randn(b, nq, t, d, device="cuda")  # (B, nh, T, d) contiguous: Liger copies, rotates the copy
    k0 = torch.randn(b, nk, t, d, device="cuda")
    cos_np, sin_np = liger_ref.rope_tables(t, d, batch=b)
    cos_np[1] = np.roll(cos_np[1], 3, axis=0)
    sin_np[1] = np.roll(sin_np[1], 3, axis=0)
    qo, ko = lk.liger_rotary_pos_emb(q0, k0, cuda(cos_np), cuda(sin_np))
    rq, rk = liger_ref.rope(q0.double().cpu().numpy(), k0.double().cpu().numpy(), cos_np, sin_np)
    assert rel_close(qo.cpu().numpy(), rq, 1e-4)[0]
    assert rel_close(ko.cpu().numpy(), rk, 1e-4)[0]


# ---------------------------------------------------------------------- GLU
@pytest.mark.parametrize("kind", ["swiglu", "geglu"])
def test_glu_fp32_vs_reference_golden(golden, kind):
    x1 = cuda(golden["glu_x1"]).requires_grad_(True)
    x2 = cuda(golden["glu_x2"]).requires_grad_(True)
    fn = lk.liger_swiglu if kind == "swiglu" else lk.liger_geglu
    y = fn(x1 * 1.0, x2 * 1.0)
    y.backward(cuda(golden["glu_dy"]))
    assert rel_close(y.detach().cpu().numpy(), golden[f"{kind}_y"], 1e-4)[0]
    assert rel_close(x1.grad.cpu().numpy(), golden[f"{kind}_dx1"], 1e-4)[0]
    assert rel_close(x2.grad.cpu().numpy(), golden[f"{kind}_dx2"], 1e-4)[0]


@pytest.mark.parametrize("kind", ["swiglu", "geglu"])
def test_glu_bf16_llama_shape(kind):
    rows, cols = 8192, 14336
    g = torch.Generator(device="cuda").manual_seed(2)
    a = (torch.randn(rows, cols, device="cuda", generator=g) * 2).to(torch.bfloat16)
    b = torch.randn(rows, cols, device="cuda", generator=g).to(torch.bfloat16)
    dc = torch.randn(rows, cols, device="cuda", generator=g).to(torch.bfloat16)
    ar, br = a.clone().requires_grad_(True), b.clone().requires_grad_(True)
    fn = lk.liger_swiglu if kind == "swiglu" else lk.liger_geglu
    c = fn(ar * 1, br * 1)
    c.backward(dc)
    sel = slice(0, 256)
    x1, x2, dy = (t[sel].double().cpu().numpy() for t in (a, b, dc))
    fwd = rp.swiglu_forward if kind == "swiglu" else rp.geglu_forward
    bwd = rp.swiglu_backward if kind == "swiglu" else rp.geglu_backward
    assert rel_close(c[sel].float().detach().cpu().numpy(), fwd(x1, x2), 2e-2)[0]
    rda, rdb = bwd(dy, x1, x2)
    assert rel_close(ar.grad[sel].float().cpu().numpy(), rda, 2e-2)[0]
    assert rel_close(br.grad[sel].float().cpu().numpy(), rdb, 2e-2)[0]


def test_swiglu_mlp_module_matches_torch():
    class Cfg:
        hidden_size, intermediate_size, hidden_act = 256, 704, "silu"

    torch.manual_seed(0)
    m = lk.LigerSwiGLUMLP(Cfg()).cuda()
    x = torch.randn(64, 256, device="cuda", requires_grad=True)
    y = m(x)
    ref = m.down_proj(torch.nn.functional.silu(m.gate_proj(x)) * m.up_proj(x))
    torch.testing.assert_close(y, ref, rtol=1e-4, atol=1e-5)
    gy = torch.randn_like(y)
    gx = torch.autograd.grad(y, x, gy)[0]
    gx_ref = torch.autograd.grad(ref, x, gy)[0]
    torch.testing.assert_close(gx, gx_ref, rtol=1e-4, atol=1e-5)


def test_benchrecord_gpu_rows(tmp_path):
    """One GPU record per op at a reference default shape, readable back through the schema."""
    from paper_2410_10989_b200 import benchrecord as br

    recs = [br.bench_op(op, *br.default_shapes(op)[0], repeats=3) for op in br.OPS]
    p = tmp_path / "gpu.csv"
    br.write_records(p, recs)
    back = br.read_records(p)
    assert [r.op for r in back] == list(br.OPS)
    assert all(r.variant == "fused" and r.median_s > 0 and r.q20_s <= r.q80_s for r in back)


def test_empty_inputs_all_ops():
    """Zero rows / tokens through every op (SURVEY §8(c) edge cases): no launch errors, empty
    outputs, zero parameter gradients."""
    dev = "cuda"
    bf = torch.bfloat16
    # RMSNorm / LayerNorm
    x = torch.empty(0, 64, dtype=bf, device=dev, requires_grad=True)
    w = torch.ones(64, dtype=bf, device=dev, requires_grad=True)
    b = torch.zeros(64, dtype=bf, device=dev, requires_grad=True)
    y = lk.liger_rms_norm(x, w, 1e-6, 0.0, "llama", False)
    y.backward(torch.empty_like(y))
    assert y.shape == (0, 64) and torch.all(w.grad == 0)
    w.grad = None
    y = lk.liger_layer_norm(x, w, b, 1e-6)
    y.backward(torch.empty_like(y))
    assert y.shape == (0, 64) and torch.all(w.grad == 0) and torch.all(b.grad == 0)
    # SwiGLU
    a = torch.empty(0, 128, dtype=bf, device=dev, requires_grad=True)
    c = lk.LigerSiLUMulFunction.apply(a, a.detach().clone().requires_grad_(True))
    assert c.shape == (0, 128)
    # RoPE with zero tokens
    q = torch.empty(1, 2, 0, 8, dtype=bf, device=dev)
    cos = torch.empty(1, 0, 8, dtype=bf, device=dev)
    qo, ko = lk.liger_rotary_pos_emb(q, q.clone(), cos, cos)
    assert qo.shape == (1, 2, 0, 8)
    # CE / FLCE with zero tokens
    z = torch.empty(0, 100, dtype=bf, device=dev, requires_grad=True)
    t = torch.empty(0, dtype=torch.long, device=dev)
    loss = lk.LigerCrossEntropyLoss(reduction="sum")(z, t)
    assert loss.item() == 0.0
    xw = torch.empty(0, 64, dtype=bf, device=dev, requires_grad=True)
    W = torch.randn(100, 64, dtype=bf, device=dev, requires_grad=True)
    loss = lk.LigerFusedLinearCrossEntropyLoss(reduction="sum")(W, xw, t)
    loss.backward()
    assert loss.item() == 0.0 and torch.all(W.grad == 0)


@pytest.mark.parametrize("kind", ["swiglu", "geglu"])
def test_glu_fp16_vs_oracle(kind):
    g = torch.Generator(device="cuda").manual_seed(61)
    a = (torch.rand(300, 1000, device="cuda", generator=g) * 8 - 4).to(torch.float16)
    b = (torch.rand(300, 1000, device="cuda", generator=g) * 2 - 1).to(torch.float16)
    dc = (torch.rand(300, 1000, device="cuda", generator=g) * 2 - 1).to(torch.float16)
    f = lk.LigerSiLUMulFunction if kind == "swiglu" else lk.LigerGELUMulFunction
    ar, br = a.clone().requires_grad_(True), b.clone().requires_grad_(True)
    c = f.apply(ar, br)
    c.backward(dc)
    fwd = rp.swiglu_forward if kind == "swiglu" else rp.geglu_forward
    bwd = rp.swiglu_backward if kind == "swiglu" else rp.geglu_backward
    a64, b64, dc64 = a.double().cpu().numpy(), b.double().cpu().numpy(), dc.double().cpu().numpy()
    rda, rdb = bwd(dc64, a64, b64)
    for name, got, ref in (("c", c.detach(), fwd(a64, b64)), ("da", ar.grad, rda), ("db", br.grad, rdb)):
        ok, err = rel_close(got.float().cpu().numpy(), ref, 2e-2)
        assert ok, (name, err)


@pytest.mark.parametrize("cols", [8192, 16384, 24576])
def test_norms_wide_rows_vs_torch(cols):
    """Wide hidden sizes: the VPT-8 CTA kernels, their launch bounds, and the fallbacks past them."""
    rows = 96
    g = torch.Generator(device="cuda").manual_seed(cols)
    x = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = (torch.rand(cols, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
    b = (torch.rand(cols, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    dy = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    xr, wr = x.clone().requires_grad_(True), w.clone().requires_grad_(True)
    lk.liger_rms_norm(xr, wr, 1e-6, 0.0, "llama", False).backward(dy)
    xf, wf = x.float().requires_grad_(True), w.float().requires_grad_(True)
    (xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + 1e-6) * wf).backward(dy.float())
    assert close(xr.grad, xf.grad, 2e-2) and close(wr.grad, wf.grad, 2e-2)
    # LayerNorm: register/TMA-ring kernels up to 16384 columns, the generic kernels beyond
    xr, wr, br = x.clone().requires_grad_(True), w.clone().requires_grad_(True), b.clone().requires_grad_(True)
    y = lk.liger_layer_norm(xr, wr, br, 1e-6)
    y.backward(dy)
    xf, wf, bf = x.float().requires_grad_(True), w.float().requires_grad_(True), b.float().requires_grad_(True)
    yf = torch.nn.functional.layer_norm(xf, (cols,), wf, bf, eps=1e-6)
    yf.backward(dy.float())
    assert close(y, yf, 2e-2) and close(xr.grad, xf.grad, 2e-2)
    assert close(wr.grad, wf.grad, 2e-2) and close(br.grad, bf.grad, 2e-2)


def test_norm_backward_in_cuda_graph():
    """The column sums are a programmatic dependent launch: they must capture and replay in a CUDA graph."""
    rows, cols = 1024, 4096
    g = torch.Generator(device="cuda").manual_seed(11)
    x = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = (torch.rand(cols, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
    b = (torch.rand(cols, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    dy = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    xs = x.clone().requires_grad_(True)
    ws, bs = w.clone().requires_grad_(True), b.clone().requires_grad_(True)

    def step():
        xs.grad = ws.grad = bs.grad = None
        lk.liger_rms_norm(xs, ws, 1e-6, 0.0, "llama", False).backward(dy)
        gx, gw = xs.grad.clone(), ws.grad.clone()
        xs.grad = None
        lk.liger_layer_norm(xs, ws, bs, 1e-6).backward(dy)
        return gx, gw, xs.grad.clone(), ws.grad.clone(), bs.grad.clone()

    eager = step()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # warm-up on the side stream (allocator pools)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = step()
    graph.replay()
    torch.cuda.synchronize()
    assert all(torch.equal(a, b_) for a, b_ in zip(eager, out))


@pytest.mark.parametrize("b,t,nq,nk,d,dtype,per_batch", [
    (3, 37, 4, 4, 64, torch.bfloat16, False),   # token-major kernel, CTA token ranges crossing sequences
    (2, 50, 6, 2, 64, torch.float32, True),     # token-major, per-batch cos/sin rows
    (5, 7, 3, 1, 128, torch.float16, False),    # 64 items per token, odd token count
    (2, 9, 3, 2, 48, torch.bfloat16, False),    # items per token not a warp multiple: grid-stride kernel
])
def test_rope_all_tokens_vs_torch(b, t, nq, nk, d, dtype, per_batch):
    g = torch.Generator(device="cuda").manual_seed(b * 1000 + t)
    q0 = torch.randn(b, t, nq, d, device="cuda", generator=g).to(dtype)
    k0 = torch.randn(b, t, nk, d, device="cuda", generator=g).to(dtype)
    ang = torch.rand(b if per_batch else 1, t, d // 2, device="cuda", generator=g) * 6.0
    emb = torch.cat([ang, ang], -1)
    cos, sin = emb.cos().to(dtype), emb.sin().to(dtype)

    def rot(x, c, s, sign):  # x (B, T, nh, d); tables (B|1, T, d)
        c, s = c[:, :, None].float(), s[:, :, None].float() * sign
        h = x.shape[-1] // 2
        xf = x.float()
        return xf * c + torch.cat([-xf[..., h:], xf[..., :h]], -1) * s

    qo, ko = lk.liger_rotary_pos_emb(q0.clone().transpose(1, 2), k0.clone().transpose(1, 2), cos, sin)
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    assert close(qo.transpose(1, 2), rot(q0, cos, sin, 1.0), tol)
    assert close(ko.transpose(1, 2), rot(k0, cos, sin, 1.0), tol)
    dq, dk, _, _ = lk.rope._rope(q0.clone().transpose(1, 2), k0.clone().transpose(1, 2), cos, sin, backward=True)
    assert close(dq.transpose(1, 2), rot(q0, cos, sin, -1.0), tol)
    assert close(dk.transpose(1, 2), rot(k0, cos, sin, -1.0), tol)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("gm,dm", [(0.7, 1.0), (2.5, 1.5), (1.0, 0.5)])
def test_swiglu_gate_and_down_multipliers(dtype, gm, dm):
    """LigerSiLUMulFunction(a, b, gate_multiplier, down_multiplier) (LK/ops/swiglu.py:16-62, 110-160)
    vs torch autograd of silu(gm * a).to(dtype) * b * dm in fp32."""
    g = torch.Generator(device="cuda").manual_seed(int(gm * 10 + dm))
    a = (torch.randn(96, 1000, device="cuda", generator=g) * 2).to(dtype)
    b = torch.randn(96, 1000, device="cuda", generator=g).to(dtype)
    dc = torch.randn(96, 1000, device="cuda", generator=g).to(dtype)
    ar, br = a.clone().requires_grad_(True), b.clone().requires_grad_(True)
    c = lk.LigerSiLUMulFunction.apply(ar, br, gm, dm)
    c.backward(dc)
    af, bf = a.float().requires_grad_(True), b.float().requires_grad_(True)
    act = torch.nn.functional.silu(gm * af)
    cf = (act.to(dtype).float() if dtype != torch.float32 else act) * bf * dm
    cf.backward(dc.float())
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    assert close(c, cf, tol)
    assert close(ar.grad, af.grad, tol) and close(br.grad, bf.grad, tol)


@pytest.mark.parametrize("cols,dtype,offset", [(1001, torch.bfloat16, 0), (4096, torch.float16, 1), (77, torch.float32, 3)])
def test_layernorm_ragged_and_unaligned_vs_torch(cols, dtype, offset):
    """Hidden sizes that are not a 16-byte multiple and storage offsets that break 16-byte
    alignment take the generic LayerNorm kernels (Liger's Triton LayerNorm takes any shape)."""
    rows = 130
    g = torch.Generator(device="cuda").manual_seed(cols + offset)
    base = (torch.rand(rows * cols + offset, device="cuda", generator=g) * 2 - 0.5).to(dtype)
    x = base[offset:].view(rows, cols)
    w = (torch.rand(cols, device="cuda", generator=g) + 0.5).to(dtype)
    b = (torch.rand(cols, device="cuda", generator=g) - 0.5).to(dtype)
    dbase = (torch.rand(rows * cols + offset, device="cuda", generator=g) * 2 - 1).to(dtype)
    dy = dbase[offset:].view(rows, cols)
    xr, wr, br = x.clone().requires_grad_(True), w.clone().requires_grad_(True), b.clone().requires_grad_(True)
    y = lk.LigerLayerNormFunction.apply(x, wr, br, 1e-6)  # x itself: the storage offset reaches the kernel
    y.backward(dy)
    xf, wf, bf = x.float().requires_grad_(True), w.float().requires_grad_(True), b.float().requires_grad_(True)
    yf = torch.nn.functional.layer_norm(xf, (cols,), wf, bf, eps=1e-6)
    yf.backward(dy.float())
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    assert close(y, yf, tol)
    assert close(wr.grad, wf.grad, tol) and close(br.grad, bf.grad, tol)



@pytest.mark.parametrize("kind", ["swiglu", "geglu"])
def test_glu_unaligned_views_vs_torch(kind):
    """Buffers whose storage offset breaks 16-byte alignment take the scalar loop of the GLU
    kernels (Liger accepts any contiguous tensor)."""
    n = 300 * 1001
    g = torch.Generator(device="cuda").manual_seed(9)
    ab = torch.randn(n + 3, device="cuda", generator=g).to(torch.bfloat16)
    bb = torch.randn(n + 5, device="cuda", generator=g).to(torch.bfloat16)
    a, b = ab[3:].view(300, 1001), bb[5:].view(300, 1001)
    dc = torch.randn(300, 1001, device="cuda", generator=g).to(torch.bfloat16)
    f = lk.LigerSiLUMulFunction if kind == "swiglu" else lk.LigerGELUMulFunction
    ar, br = ab.clone()[3:].view(300, 1001).requires_grad_(True), bb.clone()[5:].view(300, 1001).requires_grad_(True)
    c = f.apply(ar, br)
    c.backward(dc)
    af, bf = a.float().requires_grad_(True), b.float().requires_grad_(True)
    act = torch.nn.functional.silu(af) if kind == "swiglu" else torch.nn.functional.gelu(af, approximate="tanh")
    cf = act.to(torch.bfloat16).float() * bf
    cf.backward(dc.float())
    assert close(c, cf, 2e-2) and close(ar.grad, af.grad, 2e-2) and close(br.grad, bf.grad, 2e-2)


@pytest.mark.parametrize("mode", ["llama", "gemma"])
def test_rmsnorm_unaligned_views_vs_torch(mode):
    """A storage offset that breaks 16-byte alignment falls through to the generic RMSNorm kernels."""
    rows, cols = 64, 2048
    g = torch.Generator(device="cuda").manual_seed(21)
    xb = torch.randn(rows * cols + 1, device="cuda", generator=g).to(torch.bfloat16)
    dyb = torch.randn(rows * cols + 1, device="cuda", generator=g).to(torch.bfloat16)
    x, dy = xb[1:].view(rows, cols), dyb[1:].view(rows, cols)
    w = (torch.rand(cols, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
    off = 0.0 if mode == "llama" else 1.0
    xr = xb.clone()[1:].view(rows, cols).requires_grad_(True)
    wr = w.clone().requires_grad_(True)
    y = lk.liger_rms_norm(xr, wr, 1e-6, off, mode, False)
    y.backward(dy)
    xf, wf = x.float().requires_grad_(True), w.float().requires_grad_(True)
    yf = xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + 1e-6) * (off + wf)
    yf.backward(dy.float())
    assert close(y, yf, 2e-2) and close(xr.grad, xf.grad, 2e-2) and close(wr.grad, wf.grad, 2e-2)


@pytest.mark.parametrize("xdt,wdt", [(torch.bfloat16, torch.float32), (torch.float32, torch.bfloat16),
                                     (torch.float16, torch.float32)])
@pytest.mark.parametrize("mode", ["llama", "gemma"])
def test_rmsnorm_weight_dtype_differs_from_input(xdt, wdt, mode):
    """A weight whose dtype differs from X (Liger accepts an fp32 weight with bf16 activations):
    the weight is read in X's dtype and dW comes back in the weight's dtype."""
    rows, cols = 300, 1000
    g = torch.Generator(device="cuda").manual_seed(7)
    x = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(xdt)
    w = (torch.rand(cols, device="cuda", generator=g) + 0.5).to(wdt)
    dy = (torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1).to(xdt)
    offset = 1.0 if mode == "gemma" else 0.0
    xr, wr = x.clone().requires_grad_(True), w.clone().requires_grad_(True)
    y = lk.liger_rms_norm(xr, wr, 1e-6, offset, mode, False)
    y.backward(dy)
    assert y.dtype == xdt and xr.grad.dtype == xdt and wr.grad.dtype == wdt
    wq = w.to(xdt).double().cpu().numpy()  # the weight as the kernels read it
    ry, _ = liger_ref.rmsnorm_fwd(x.double().cpu().numpy(), wq, 1e-6, offset)
    rdx, _ = liger_ref.rmsnorm_bwd(dy.double().cpu().numpy(), x.double().cpu().numpy(), wq, 1e-6, offset)
    assert rel_close(y.float().detach().cpu().numpy(), ry, 2e-2)[0]
    assert rel_close(xr.grad.float().cpu().numpy(), rdx, 2e-2)[0]
    xf, dyf = x.double(), dy.double()
    rdw = (dyf * xf * torch.rsqrt((xf * xf).mean(1, keepdim=True) + 1e-6)).sum(0)
    assert close(wr.grad.double(), rdw, 2e-2)
