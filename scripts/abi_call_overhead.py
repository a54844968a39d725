"""Host cost of individual C-ABI calls (no sync in the loop).  python scripts/abi_call_overhead.py"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2410_10989_b200 as lk
from paper_2410_10989_b200._utils import lib, stream_of, ptr, dtype_code

L = lib()
dev = torch.device("cuda")
x = torch.randn(8192, 4096, device=dev, dtype=torch.bfloat16)
w = torch.ones(4096, device=dev, dtype=torch.bfloat16)
y = torch.empty_like(x)
r = torch.empty(8192, device=dev)
st = stream_of(x)


def t(name, fn, n=2000):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    print(f"{name}: {dt:.2f} us")


t("lk_has_tcgen05", lambda: L.lk_has_tcgen05())
t("stream_of", lambda: stream_of(x))
t("lk_rmsnorm_fwd (8192x4096)", lambda: L.lk_rmsnorm_fwd(x.data_ptr(), w.data_ptr(), y.data_ptr(), r.data_ptr(), 8192,
                                                          4096, 1e-6, 0.0, 1, dtype_code(x), st), n=200)
t("torch add_ (8192x4096)", lambda: y.add_(x), n=200)
t("torch.empty_like", lambda: torch.empty_like(x))
t("torch.cuda.device ctx", lambda: torch.cuda.device(0).__enter__())

from paper_2410_10989_b200.rms_norm import rms_norm_forward, rms_norm_backward
t("rms_norm_forward()", lambda: rms_norm_forward(x, w, 1e-6), n=200)
Y, X2, rstd, mode = rms_norm_forward(x, w, 1e-6)
dy = torch.randn_like(x)
t("rms_norm_backward() (not in place)", lambda: rms_norm_backward(dy, X2, w, rstd, 0.0, mode, False), n=200)
wp = torch.nn.Parameter(w.clone())
def fb():
    xx = x.detach().requires_grad_(True)
    lk.liger_rms_norm(xx, wp, 1e-6, 0.0, "llama", False).backward(dy)
t("liger_rms_norm fwd+bwd autograd", fb, n=200)
ws = torch.empty(L.lk_rmsnorm_bwd_workspace_bytes(8192, 4096), dtype=torch.uint8, device=dev)
dx = torch.empty_like(x); dw = torch.empty_like(w)
t("lk_rmsnorm_bwd raw", lambda: L.lk_rmsnorm_bwd(dy.data_ptr(), x.data_ptr(), w.data_ptr(), r.data_ptr(), dx.data_ptr(),
                                                  dw.data_ptr(), 8192, 4096, 0.0, 1, dtype_code(x), ws.data_ptr(),
                                                  ws.numel(), st), n=200)
