"""Tensor-pipe efficiency of the CTA-pair tcgen05 GEMM versus tile length, at equal FLOPs (GPU).

    python scripts/gemm_shape_probe.py
Shapes: one long tile per CTA pair (74 tiles of 2048 k-blocks: no tile switches) down to many
short tiles.  bf16 store epilogue (lk_gemm_test_accum16, beta = 0).  TFLOP/s over the median
of 5 launches; nvidia-smi clocks are not sampled, so compare shapes within one run."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2410_10989_b200 import _capi  # noqa: E402

L = _capi.load()
dev = torch.device("cuda")
ws = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
M = 74 * 256
SHAPES = [(256, 131072), (1024, 32768), (4096, 8192), (16384, 2048), (32768, 1024)]


def time_shape(n, k, reps=5):
    a = (torch.rand(M, k, device=dev) - 0.5).to(torch.bfloat16)
    b = (torch.rand(n, k, device=dev) - 0.5).to(torch.bfloat16)
    d = torch.empty(M, n, dtype=torch.bfloat16, device=dev)
    call = lambda: L.lk_gemm_test_accum16(a.data_ptr(), b.data_ptr(), d.data_ptr(), M, n, k, _capi.LK_BF16, 0, 1,  # noqa: E731
                                          ws.data_ptr(), ws.numel(), st)
    assert call() == 0
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]


res = {s: [] for s in SHAPES}
for _ in range(3):
    for s in SHAPES:
        res[s].append(time_shape(*s))


def time_cublas(n, k, reps=5):
    a = (torch.rand(M, k, device=dev) - 0.5).to(torch.bfloat16)
    b = (torch.rand(n, k, device=dev) - 0.5).to(torch.bfloat16)
    torch.matmul(a, b.t())
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b.t())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]


cub = {s: [] for s in SHAPES}
for _ in range(3):
    for s in SHAPES:
        cub[s].append(time_cublas(*s))
        res[s].append(time_shape(*s))  # interleaved with cuBLAS: same clock state
for (n, k), ts in res.items():
    ms, mc = min(ts), min(cub[(n, k)])
    tiles = (M // 256) * (n // 256)
    print(json.dumps({"N": n, "K": k, "tiles": tiles, "k_blocks_per_tile": k // 64, "ms": round(ms, 4),
                      "tflops": round(2 * M * n * k / (ms / 1e3) / 1e12, 1),
                      "cublas_tflops": round(2 * M * n * k / (mc / 1e3) / 1e12, 1)}), flush=True)
