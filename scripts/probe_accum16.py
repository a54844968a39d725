import sys, torch
sys.path.insert(0, ".")
from paper_2410_10989_b200 import _capi
lib = _capi.load()
g = torch.Generator(device="cuda").manual_seed(5)
m, n, k = 512, 512, 256
a1 = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
b1 = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
a2 = (torch.randn(m, k, device="cuda", generator=g) * 0.37).to(torch.bfloat16)
b2 = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
ws = torch.empty(256, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for tma in (1, 0):
    d = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    for beta, (a, b) in enumerate(((a1, b1), (a2, b2))):
        _capi.check(lib.lk_gemm_test_accum16(a.data_ptr(), b.data_ptr(), d.data_ptr(), m, n, k, 1, beta, tma, ws.data_ptr(), ws.numel(), st))
        torch.cuda.synchronize()
        if beta == 0:
            p1got = d.float().clone()
    p1 = (a1.float() @ b1.float().T)
    p2 = a2.float() @ b2.float().T
    print("tma", tma, "first store == bf16(p1):", (p1got == p1.to(torch.bfloat16).float()).float().mean().item())
    for name, want in (("rn(acc+rn(p2))", (p1got + p2.to(torch.bfloat16).float()).to(torch.bfloat16).float()),
                       ("rn(acc+p2)", (p1got + p2).to(torch.bfloat16).float()),
                       ("trunc(acc+rn(p2))", ((p1got + p2.to(torch.bfloat16).float()).view(torch.int32) & ~0xffff).view(torch.float32))):
        got = d.float()
        bad = (got != want)
        diff = (got - want).abs()
        print(f"  {name}: equal {1 - bad.float().mean().item():.4f} maxdiff {diff.max().item():.4g} rel-to-ulp {(diff / (want.abs() * 2**-8 + 1e-30)).max().item():.3g}")
        if name == "rn(acc+rn(p2))":
            idx = bad.nonzero()[:10].tolist()
            print("   first bad", idx, [(got[i, j].item(), want[i, j].item(), p1got[i, j].item(), p2[i, j].item()) for i, j in idx[:4]])
