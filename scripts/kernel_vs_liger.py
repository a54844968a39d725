"""Kernel-level steady-state comparison with upstream Liger-Kernel 0.8.0 (Triton) on one B200.

Both implementations are called at the op level, with no autograd: ours through the C ABI,
Liger through `liger_kernel.ops.*`. Each implementation cycles over 4 independent buffer
sets whose combined size exceeds the 126 MB L2, back to back, captured in one CUDA graph so
host launch cost is out of the loop. Reported: GPU time per call and the fraction of the
measured HBM bandwidth for the same algorithmic bytes as `bench_kernels.py`.

    python scripts/kernel_vs_liger.py [--reps 20]
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import measured_peaks  # noqa: E402
from paper_2410_10989_b200 import _capi  # noqa: E402

BT, H, I, NQ, NK, D = 8192, 4096, 14336, 32, 8, 128


def graph_time(fns, reps):
    """ms per call: `reps` rounds over `fns` in one captured graph, median of 3 replays."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fns:
            f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            for f in fns:
                f()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / (reps * len(fns)))
    del g
    return sorted(ts)[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="rope,rmsnorm,layernorm,swiglu")
    args = ap.parse_args()
    want = set(args.only.split(","))
    from liger_kernel.ops import layer_norm as ULN
    from liger_kernel.ops import rms_norm as URMS
    from liger_kernel.ops import rope as UROPE
    from liger_kernel.ops import swiglu as USW

    L = _capi.load()
    dev = torch.device("cuda")
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    bf = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(0)
    hbm = float(measured_peaks()[0]["hbm_gbs"])
    out = []

    def report(op, nbytes, ours_ms, liger_ms):
        rec = {"op": op, "bytes": nbytes, "b200_us": round(ours_ms * 1e3, 2), "liger_us": round(liger_ms * 1e3, 2),
               "b200_frac": round(nbytes / (ours_ms / 1e3) / 1e9 / hbm, 3),
               "liger_frac": round(nbytes / (liger_ms / 1e3) / 1e9 / hbm, 3),
               "speedup": round(liger_ms / ours_ms, 3)}
        out.append(rec)
        print(json.dumps(rec), flush=True)

    # ---- RoPE: q (B, T, 32, 128), k (B, T, 8, 128), in place, physical (B, T, H, D) ----
    B, T = 4, 2048
    w = (torch.rand(H, device=dev, generator=g) + 0.5).to(bf)
    dw = torch.empty_like(w)
    ang = torch.rand(1, T, D, device=dev, generator=g) * 6.28
    cos, sin = torch.cos(ang).to(bf), torch.sin(ang).to(bf)
    sets = [(torch.randn(B, T, NQ, D, device=dev, generator=g).to(bf),
             torch.randn(B, T, NK, D, device=dev, generator=g).to(bf)) for _ in range(4)] if "rope" in want else []
    nbytes = 2 * (B * T * (NQ + NK) * D) * 2 + 2 * T * (D // 2) * 2
    for bwd, name in ((0, "rope_fwd"), (1, "rope_bwd")) if "rope" in want else ():
        ours = [lambda q=q, k=k, b=bwd: L.lk_rope(q.data_ptr(), k.data_ptr(), cos.data_ptr(), sin.data_ptr(), B, T, NQ,
                                                  NK, D, 1, 1, 1, b, st()) for q, k in sets]
        uf = UROPE.rope_backward if bwd else UROPE.rope_forward
        up = [lambda q=q, k=k, f=uf: f(q.transpose(1, 2), k.transpose(1, 2), cos, sin) for q, k in sets]
        report(name, nbytes, graph_time(ours, args.reps), graph_time(up, args.reps))
    del sets

    if "rmsnorm" in want:
        # ---- RMSNorm (llama casting, offset 0) ----
        ws = torch.empty(L.lk_rmsnorm_bwd_workspace_bytes(BT, H), dtype=torch.uint8, device=dev)
        sets = []
        for _ in range(4):
            x = torch.randn(BT, H, device=dev, generator=g).to(bf)
            sets.append(dict(x=x, y=torch.empty_like(x), rstd=torch.empty(BT, device=dev),
                             dy=torch.randn(BT, H, device=dev, generator=g).to(bf), dx=torch.empty_like(x)))
        ours = [lambda d=d: L.lk_rmsnorm_fwd(d["x"].data_ptr(), w.data_ptr(), d["y"].data_ptr(), d["rstd"].data_ptr(), BT,
                                             H, 1e-6, 0.0, 0, 1, st()) for d in sets]
        up = [lambda d=d: URMS.rms_norm_forward(d["x"], w, 1e-6, 0.0, "llama", None) for d in sets]
        report("rmsnorm_fwd", 2 * BT * H * 2 + H * 2 + BT * 4, graph_time(ours, args.reps), graph_time(up, args.reps))
        ulr = [URMS.rms_norm_forward(d["x"], w, 1e-6, 0.0, "llama", None) for d in sets]  # (Y, X, RSTD, BS, nw, mode)
        for d in sets:
            L.lk_rmsnorm_fwd(d["x"].data_ptr(), w.data_ptr(), d["y"].data_ptr(), d["rstd"].data_ptr(), BT, H, 1e-6, 0.0, 0,
                             1, st())
        ours = [lambda d=d: L.lk_rmsnorm_bwd(d["dy"].data_ptr(), d["x"].data_ptr(), w.data_ptr(), d["rstd"].data_ptr(),
                                             d["dx"].data_ptr(), dw.data_ptr(), BT, H, 0.0, 0, 1, ws.data_ptr(), ws.numel(),
                                             st()) for d in sets]
        up = [lambda d=d, r=r: URMS.rms_norm_backward(d["dy"], r[1], w, r[2], 0.0, r[5], r[3], r[4], False, None)
              for d, r in zip(sets, ulr)]
        report("rmsnorm_bwd", 3 * BT * H * 2 + H * 2 * 2 + BT * 4, graph_time(ours, args.reps), graph_time(up, args.reps))
        del sets, ulr

    if "layernorm" in want:
        # ---- LayerNorm ----
        b = torch.randn(H, device=dev, generator=g).to(bf)
        db = torch.empty_like(b)
        lws = torch.empty(L.lk_layernorm_bwd_workspace_bytes(BT, H), dtype=torch.uint8, device=dev)
        sets = []
        for _ in range(4):
            x = torch.randn(BT, H, device=dev, generator=g).to(bf)
            sets.append(dict(x=x, y=torch.empty_like(x), dy=torch.randn(BT, H, device=dev, generator=g).to(bf),
                             dx=torch.empty_like(x), mu=torch.empty(BT, device=dev), rs=torch.empty(BT, device=dev)))
        ours = [lambda d=d: L.lk_layernorm_fwd(d["x"].data_ptr(), w.data_ptr(), b.data_ptr(), d["y"].data_ptr(),
                                               d["mu"].data_ptr(), d["rs"].data_ptr(), BT, H, 1e-6, 1, st()) for d in sets]
        up = [lambda d=d: ULN.layer_norm_forward(d["x"], w, b, 1e-6) for d in sets]
        report("layernorm_fwd", 2 * BT * H * 2 + 2 * H * 2 + 2 * BT * 4, graph_time(ours, args.reps),
               graph_time(up, args.reps))
        ulf = [ULN.layer_norm_forward(d["x"], w, b, 1e-6) for d in sets]  # (Y, X, Mean, RSTD, BS, nw)
        for f in ours:
            f()
        ours = [lambda d=d: L.lk_layernorm_bwd(d["dy"].data_ptr(), d["x"].data_ptr(), w.data_ptr(), d["mu"].data_ptr(),
                                               d["rs"].data_ptr(), d["dx"].data_ptr(), dw.data_ptr(), db.data_ptr(), BT, H,
                                               1, lws.data_ptr(), lws.numel(), st()) for d in sets]
        up = [lambda d=d, r=r: ULN.layer_norm_backward(d["dy"], r[1], w, b, r[2], r[3]) for d, r in zip(sets, ulf)]
        report("layernorm_bwd", 3 * BT * H * 2 + 3 * H * 2 + 2 * BT * 4, graph_time(ours, args.reps),
               graph_time(up, args.reps))
        del sets, ulf

    if "swiglu" in want:
        # ---- SwiGLU (8192 x 14336) ----
        n = BT * I
        sets = [dict(a=torch.randn(BT, I, device=dev, generator=g).to(bf), b=torch.randn(BT, I, device=dev, generator=g).to(bf),
                     c=torch.empty(BT, I, device=dev, dtype=bf),
                     dc=(torch.randn(BT, I, device=dev, generator=g) * 1e-3).to(bf)) for _ in range(2)]
        ours = [lambda d=d: L.lk_swiglu_fwd(d["a"].data_ptr(), d["b"].data_ptr(), d["c"].data_ptr(), n, 1, st())
                for d in sets]
        up = [lambda d=d: USW.swiglu_forward(d["a"], d["b"]) for d in sets]
        report("swiglu_fwd", 3 * n * 2, graph_time(ours, args.reps), graph_time(up, args.reps))
        ours = [lambda d=d: L.lk_swiglu_bwd(d["dc"].data_ptr(), d["a"].data_ptr(), d["b"].data_ptr(), n, 1, st())
                for d in sets]
        up = [lambda d=d: USW.swiglu_backward(d["a"], d["b"], d["dc"]) for d in sets]
        report("swiglu_bwd", 5 * n * 2, graph_time(ours, args.reps), graph_time(up, args.reps))
    print(json.dumps({"summary": {r["op"]: r["speedup"] for r in out}}), flush=True)


if __name__ == "__main__":
    main()
