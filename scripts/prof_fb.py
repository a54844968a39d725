import sys, cProfile, pstats
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2410_10989_b200 as lk
dev = torch.device("cuda")
x = torch.randn(8192, 4096, device=dev, dtype=torch.bfloat16)
dy = torch.randn_like(x)
wp = torch.nn.Parameter(torch.ones(4096, device=dev, dtype=torch.bfloat16))
def fb():
    xx = x.detach().requires_grad_(True)
    lk.liger_rms_norm(xx, wp, 1e-6, 0.0, "llama", False).backward(dy)
for _ in range(20): fb()
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(200): fb()
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
