"""Probe: tcgen05 GEMM throughput vs the K-major row stride (power-of-two camping check)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2410_10989_b200 import _capi

lib = _capi.load()
dev = torch.device("cuda")
ws = torch.empty(256, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
M, N = 2048, 32768
for K in (4096, 4160, 4032, 3584, 3648, 8192, 8256):
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    b = torch.randn(N, K, device=dev).to(torch.bfloat16)
    d = torch.empty(M, N, device=dev)
    f = lambda: _capi.check(lib.lk_gemm_test(a.data_ptr(), b.data_ptr(), d.data_ptr(), M, N, K, 0, 1, 2, ws.data_ptr(), ws.numel(), st))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"K={K} stride={K*2}B  {ms:.3f} ms  {2*M*N*K/ms/1e9:.0f} TFLOP/s")
