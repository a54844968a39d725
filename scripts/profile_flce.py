"""Short FLCE driver for ncu: cfg2 shape, a few steps (never a bench number)."""

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_10989_b200.fused_linear_cross_entropy import fused_linear_cross_entropy_forward  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--bt", type=int, default=8192)
ap.add_argument("--hidden", type=int, default=4096)
ap.add_argument("--vocab", type=int, default=128256)
ap.add_argument("--chunk-rows", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
x = (torch.rand(a.bt, a.hidden, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
w = ((torch.rand(a.vocab, a.hidden, device=dev, generator=g) * 2 - 1) / 64).to(torch.bfloat16)
t = torch.randint(0, a.vocab, (a.bt,), device=dev, generator=g)
t[torch.rand(a.bt, device=dev, generator=g) < 0.1] = -100
for _ in range(a.steps):
    fused_linear_cross_entropy_forward(x, w, t, chunk_rows=a.chunk_rows or None, compute_grad_input=True,
                                       compute_grad_weight=True)
torch.cuda.synchronize()
print("done")
