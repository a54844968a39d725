"""tcgen05 / TMA GEMM exactness for the three FLCE operand layouts (GPU).

Inputs are small integers stored in bf16, so every product and every partial
sum is exact in fp32: the tensor-core result must equal torch's fp32 matmul
bit for bit.  Any error in the smem descriptors, swizzle, instruction
descriptor or TMEM addressing shows up as a hard mismatch.
"""

import pytest
import torch

from paper_2410_10989_b200 import _capi

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 64), (256, 512, 192), (200, 264, 136), (64, 40, 520), (1000, 776, 320)]


def run(a, b, m, n, k, layout, tc):
    d = torch.full((m, n), float("nan"), device="cuda", dtype=torch.float32)
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    lib = _capi.load()
    _capi.check(lib.lk_gemm_test(a.data_ptr(), b.data_ptr(), d.data_ptr(), m, n, k, layout, 1, int(tc),
                                 ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return d


def operands(m, n, k, layout, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randint(-3, 4, (m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randint(-3, 4, (k, n), device="cuda", generator=g).to(torch.bfloat16)
    ref = A.float() @ B.float()
    if layout == 0:
        return A.contiguous(), B.t().contiguous(), ref      # A[M,K], B[N,K]
    if layout == 1:
        return A.contiguous(), B.contiguous(), ref          # A[M,K], B[K,N]
    return A.t().contiguous(), B.contiguous(), ref          # A[K,M], B[K,N]


@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("layout", [0, 1, 2])
@pytest.mark.parametrize("shape", SHAPES)
def test_tcgen05_gemm_exact(layout, shape, cta_group):
    m, n, k = shape
    if layout == 2 and m % 8:
        pytest.skip("M-major A needs M % 8 == 0 for TMA")
    a, b, ref = operands(m, n, k, layout, seed=m + n + k + layout)
    d = run(a, b, m, n, k, layout, tc=cta_group)
    bad = (d != ref).sum().item()
    assert bad == 0, f"{bad} mismatches; first at {torch.nonzero(d != ref)[:4].tolist()}"


@pytest.mark.parametrize("layout", [0, 1, 2])
def test_simt_gemm_exact(layout):
    m, n, k = 200, 264, 136
    a, b, ref = operands(m, n, k, layout, seed=7)
    d = run(a, b, m, n, k, layout, tc=False)
    assert torch.equal(d, ref)


def test_tcgen05_gemm_random_bf16_large():
    m, n, k = 2048, 4096, 4096
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
    d = run(A, B, m, n, k, 0, tc=2)
    ref = A.float() @ B.float().t()
    err = (d - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("tma_reduce", [1, 0])
def test_accum16_epilogue_rounding(tma_reduce):
    """16-bit grad_w accumulation (weight-dtype accum_dtype): store, then add a second product.
    TMA reduce-add path: the tile is staged in bf16 and added in L2 -> bf16(acc + bf16(p2)),
    exactly Liger's `grad_weight += torch.mm(...).float()` order with a bf16 grad_weight
    (LK/ops/fused_linear_cross_entropy.py:211).  Register path: bf16(acc + p2)."""
    lib = _capi.load()
    g = torch.Generator(device="cuda").manual_seed(5)
    m, n, k = 512, 512, 256
    a1 = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b1 = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
    a2 = (torch.randn(m, k, device="cuda", generator=g) * 0.37).to(torch.bfloat16)
    b2 = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
    d = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(256, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for beta, (a, b) in enumerate(((a1, b1), (a2, b2))):
        _capi.check(lib.lk_gemm_test_accum16(a.data_ptr(), b.data_ptr(), d.data_ptr(), m, n, k, 1, beta, tma_reduce,
                                             ws.data_ptr(), ws.numel(), st))
    torch.cuda.synchronize()
    p1 = (a1.float() @ b1.float().T).to(torch.bfloat16).float()
    p2 = a2.float() @ b2.float().T
    want = (p1 + (p2.to(torch.bfloat16).float() if tma_reduce else p2)).to(torch.bfloat16).float()
    got = d.float()
    # fp32 summation order inside the MMA differs from torch's, so a rounding of p1 / p2 can land
    # one ulp apart at ties: equal almost everywhere, and never more than a few bf16 ulps apart
    assert (got == want).float().mean().item() > 0.99
    ulp = torch.clamp(want.abs(), min=1e-3) * 2.0**-7
    assert torch.all((got - want).abs() <= 4 * ulp)
