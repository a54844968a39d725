"""One dW-shaped tcgen05 GEMM launch per K (warm-up first) for ncu: D[128256, 4096] += A . B^T,
bf16 TMA reduce-add epilogue (lk_gemm_test_accum16).  python scripts/dw_gemm_once.py 2560 10240"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2410_10989_b200 import _capi  # noqa: E402

L = _capi.load()
V, H = 128256, 4096
ks = [int(a) for a in sys.argv[1:]] or [2560]
dev = torch.device("cuda")
D16 = torch.zeros(V, H, dtype=torch.bfloat16, device=dev)
ws = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
for k in ks:
    a = (torch.rand(V, k, device=dev) - 0.5).to(torch.bfloat16)
    b = (torch.rand(H, k, device=dev) - 0.5).to(torch.bfloat16)
    for _ in range(2):  # warm-up launch, then the captured one
        assert L.lk_gemm_test_accum16(a.data_ptr(), b.data_ptr(), D16.data_ptr(), V, H, k, _capi.LK_BF16, 1, 1,
                                      ws.data_ptr(), ws.numel(), st) == 0
    torch.cuda.synchronize()
    del a, b
