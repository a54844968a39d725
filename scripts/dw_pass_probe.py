"""Where the per-chunk dW pass cost goes: the dW-shaped GEMM alone,
D[V=128256, H=4096] (+)= A[V, K] . B[H, K]^T on the CTA-pair tcgen05 kernel, timed at several K.

    python scripts/dw_pass_probe.py
A fit T(K) = a + b*K separates the K-proportional MMA time from the fixed cost of one pass over
the 8016 output tiles (epilogue, tile switches, launch).  Epilogues: bf16 TMA reduce-add into
D (the FLCE's middle chunks), bf16 TMA store (first chunk), fp32 store (lk_gemm_test)."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2410_10989_b200 import _capi  # noqa: E402

L = _capi.load()
V, H = 128256, 4096
KS = [1280, 2560, 5120, 10240]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
A = (torch.rand(V, max(KS), device=dev, generator=g) - 0.5).to(torch.bfloat16)
B = (torch.rand(H, max(KS), device=dev, generator=g) - 0.5).to(torch.bfloat16)
D16 = torch.zeros(V, H, dtype=torch.bfloat16, device=dev)
ws = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731


def run(k, mode):
    a = A[:, :k].contiguous() if k != max(KS) else A
    b = B[:, :k].contiguous() if k != max(KS) else B
    def call():
        if mode == "reduce16":
            return L.lk_gemm_test_accum16(a.data_ptr(), b.data_ptr(), D16.data_ptr(), V, H, k, _capi.LK_BF16, 1, 1,
                                          ws.data_ptr(), ws.numel(), st())
        return L.lk_gemm_test_accum16(a.data_ptr(), b.data_ptr(), D16.data_ptr(), V, H, k, _capi.LK_BF16, 0, 1,
                                      ws.data_ptr(), ws.numel(), st())
    assert call() == 0
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    del a, b
    return sorted(ts)[2]


res = {}
for rnd in range(2):
    for mode in ("reduce16", "store16"):
        for k in KS:
            res.setdefault((mode, k), []).append(run(k, mode))
for mode in ("reduce16", "store16"):
    pts = [(k, min(res[(mode, k)])) for k in KS]
    n = len(pts)
    mk = sum(p[0] for p in pts) / n
    mt = sum(p[1] for p in pts) / n
    b = sum((p[0] - mk) * (p[1] - mt) for p in pts) / sum((p[0] - mk) ** 2 for p in pts)
    a = mt - b * mk
    print(json.dumps({"epilogue": mode, "ms": {k: round(t, 3) for k, t in pts},
                      "fit_fixed_ms": round(a, 3), "fit_ms_per_1k_rows": round(b * 1000, 3),
                      "tflops_at_k": {k: round(2 * V * H * k / (t / 1e3) / 1e12) for k, t in pts}}), flush=True)
