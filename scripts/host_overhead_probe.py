"""Host time per FLCE call on a tiny problem (GPU time negligible), with and without the
kept-row path, plus a cProfile of the kept-row call (GPU box)."""

import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2410_10989_b200.fused_linear_cross_entropy as m  # noqa: E402

m.COMPACT_MIN_SKIPPED = 1
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(512, 256, device="cuda", generator=g).to(torch.bfloat16)
w = torch.rand(1024, 256, device="cuda", generator=g).to(torch.bfloat16)
t = torch.randint(0, 1024, (512,), device="cuda", generator=g)
t[::3] = -100
for skip in (False, True):
    kw = dict(compute_grad_input=True, compute_grad_weight=True, skip_ignored_rows=skip, check_targets=False)
    for _ in range(20):
        m.fused_linear_cross_entropy_forward(x, w, t, **kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        m.fused_linear_cross_entropy_forward(x, w, t, **kw)
        torch.cuda.synchronize()
    print(f"skip={skip}: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us per call incl. sync", flush=True)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    m.fused_linear_cross_entropy_forward(x, w, t, compute_grad_input=True, compute_grad_weight=True,
                                         skip_ignored_rows=True, check_targets=False)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
