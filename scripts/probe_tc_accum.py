"""Probe: how the tcgen05 kind::f16 fp32 accumulator rounds over long K, and what that does to
the fp32 (split-operand) FLCE at the cfg2 shape.  Prints one JSON object per probe."""

import json
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_10989_b200 import _capi  # noqa: E402
from paper_2410_10989_b200.fused_linear_cross_entropy import fused_linear_cross_entropy_forward as flce_fwd  # noqa: E402
from oracle import liger_ref  # noqa: E402  (checker)

lib = _capi.load()


def tc_gemm(A, Bt):  # A[M,K], Bt[N,K] bf16 -> fp32 D[M,N] on tcgen05 (layout 0)
    m, k = A.shape
    n = Bt.shape[0]
    d = torch.empty((m, n), device="cuda", dtype=torch.float32)
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    _capi.check(lib.lk_gemm_test(A.data_ptr(), Bt.data_ptr(), d.data_ptr(), m, n, k, 0, 1, 1, ws.data_ptr(),
                                 ws.numel(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return d


def accum_probe():
    out = {}
    for K in (64, 1024, 16384):
        for name, delta in (("0.75ulp", 0.75 * 2.0**-23), ("0.5ulp", 0.5 * 2.0**-23), ("0.25ulp", 0.25 * 2.0**-23),
                            ("2ulp", 2.0 * 2.0**-23)):
            for where in ("first", "last"):
                A = torch.full((128, K), delta, dtype=torch.float64)
                if where == "first":
                    A[:, 0] = 1.0
                else:
                    A[:, -1] = 1.0
                A = A.to(torch.bfloat16).cuda()
                Bt = torch.ones((256, K), dtype=torch.bfloat16, device="cuda")
                d = tc_gemm(A, Bt)[0, 0].item()
                exact = 1.0 + (K - 1) * float(A[0, 1 if where == "first" else 0].double())
                out[f"K{K}_{name}_{where}"] = {"tc": d, "exact": exact, "ulps_lost": (exact - d) / 2.0**-23}
    print(json.dumps({"probe": "accum_ones", **out}))
    # random long-K: error bias vs fp64
    g = torch.Generator(device="cuda").manual_seed(0)
    for K in (4096, 65536, 393216):
        A = (torch.rand(128, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        Bt = (torch.rand(256, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        d = tc_gemm(A, Bt).double()
        ref = A.double() @ Bt.double().t()
        err = d - ref
        scale = (A.double().abs() @ Bt.double().abs().t())
        print(json.dumps({"probe": "accum_random", "K": K, "max_abs_err": err.abs().max().item(),
                          "mean_err": err.mean().item(), "mean_abs_err": err.abs().mean().item(),
                          "rel_to_sum_abs": (err.abs() / scale).max().item(),
                          "rel_to_max_ref": (err.abs().max() / ref.abs().max()).item()}))


def rel(a, b):
    a = np.asarray(a, np.float64)
    scale = np.abs(b).max()
    return float((np.abs(a - b) / (np.abs(b) + scale)).max()), float(np.abs(a - b).max() / scale)


def flce_probe():
    for V in (16384, 128256):
        g = torch.Generator(device="cuda").manual_seed(5)
        x = torch.rand(256, 4096, device="cuda", generator=g) * 2 - 1
        w = (torch.rand(V, 4096, device="cuda", generator=g) * 2 - 1) / 64.0
        t = torch.randint(0, V, (256,), device="cuda", generator=g)
        t[torch.rand(256, device="cuda", generator=g) < 0.1] = -100
        ref_loss, _, _, rgx, rgw, _ = liger_ref.flce(x.double().cpu().numpy(), w.double().cpu().numpy(),
                                                     t.cpu().numpy())
        for name, kw in (("p2", dict(fp32_pieces=2)), ("p3", dict(fp32_pieces=3)), ("simt", dict(force_simt=True))):
            loss, _, _, _, gx, gw, _ = flce_fwd(x, w, t, compute_grad_input=True, compute_grad_weight=True, **kw)
            torch.cuda.synchronize()
            print(json.dumps({"probe": "flce_fp32", "V": V, "path": name,
                              "loss_rel": abs(loss.item() - ref_loss) / abs(ref_loss),
                              "dx_rel_tolform": rel(gx.cpu().numpy(), rgx)[0], "dx_err_over_max": rel(gx.cpu().numpy(), rgx)[1],
                              "dw_rel_tolform": rel(gw.cpu().numpy(), rgw)[0], "dw_err_over_max": rel(gw.cpu().numpy(), rgw)[1]}))


if __name__ == "__main__":
    accum_probe()
    flce_probe()
