"""Host-side issue time per fwd+bwd call of the small ops (no sync inside the loop): the
floor below which a short kernel's wall time cannot go.  python scripts/cpu_overhead.py"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2410_10989_b200 as lk

dev = torch.device("cuda")
bf = torch.bfloat16
x = torch.randn(8192, 4096, device=dev, dtype=bf)
dy = torch.randn(8192, 4096, device=dev, dtype=bf)
rms = lk.LigerRMSNorm(4096).to(dev, bf)
ln = lk.LigerLayerNorm(4096).to(dev, bf)
tln = torch.nn.LayerNorm(4096).to(dev, bf)


def issue_time(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) / n * 1e6, (t2 - t0) / n * 1e6


def f_rms():
    xx = x.detach().requires_grad_(True)
    rms(xx).backward(dy)


def f_ln():
    xx = x.detach().requires_grad_(True)
    ln(xx).backward(dy)


def f_tln():
    xx = x.detach().requires_grad_(True)
    tln(xx).backward(dy)


for name, fn in [("rmsnorm", f_rms), ("layernorm", f_ln), ("torch layernorm", f_tln)]:
    a, b = issue_time(fn)
    print(f"{name}: host issue {a:.1f} us/call, wall {b:.1f} us/call")
