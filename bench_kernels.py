#!/usr/bin/env python
"""Bandwidth-kernel benchmark at BASELINE cfg3 (Llama-3-8B decoder block, BT=8192, bf16).

Each kernel runs through the C ABI on device-resident inputs, two ways: `ms`/`frac` = one
launch with a cold L2 (512 MiB read between timed launches: several cfg3 operands fit the
126 MB L2), `steady_ms`/`steady_frac` = back-to-back launches cycling over 2-4 independent
buffer sets whose combined size exceeds L2 (the in-step cost, launch gaps hidden).  achieved = algorithmic bytes / CUDA-event time,
frac = achieved / measured HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs).
Prints one JSON line per kernel, and a summary line.

    python bench_kernels.py [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from bench import measured_peaks  # noqa: E402
from paper_2410_10989_b200 import _capi  # noqa: E402

BT, H, I, NQ, NK, D, V = 8192, 4096, 14336, 32, 8, 128, 128256


def timed(fn, reps, flush):
    fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        # evict L2 by READING 512 MiB (a write-based flush would leave dirty lines whose
        # write-back would be charged to the timed kernel)
        flush_sink.copy_(flush.view(torch.int64).sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    return statistics.median(times)


def steady(fns, reps):
    """Back-to-back launches cycling over independent buffer sets (each set's bytes were last
    touched len(fns)-1 launches earlier, so L2 holds none of them): in-stream cost per launch
    with launch gaps hidden, as inside a model step."""
    for f in fns:
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for f in fns:
            f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * len(fns))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    dev = torch.device("cuda")
    L = _capi.load()
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    global flush_sink
    flush = torch.ones(512 * 2**20, dtype=torch.uint8, device=dev)
    flush_sink = torch.zeros((), dtype=torch.int64, device=dev)
    peaks, src = measured_peaks()
    hbm = float(peaks["hbm_gbs"])
    bf = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(0)
    out = []

    def report(name, bytes_, ms, extra=None):
        gbs = bytes_ / (ms / 1e3) / 1e9
        line = {"kernel": name, "bytes": bytes_, "ms": ms, "achieved_gbs": gbs, "peak_gbs": hbm,
                "frac": gbs / hbm, "peak_source": f"{src} hbm_gbs", "bound": "hbm"}
        if extra:
            line.update(extra)
        out.append(line)
        print(json.dumps(line), flush=True)

    want = lambda n: (not args.only) or any(k in n for k in args.only.split(","))  # noqa: E731

    # ---- RMSNorm (x: 8192 x 4096) ----
    if want("rmsnorm"):
        sets = []
        for _ in range(4):
            x = torch.randn(BT, H, device=dev, generator=g).to(bf)
            sets.append(dict(x=x, y=torch.empty_like(x), rstd=torch.empty(BT, device=dev),
                             dy=torch.randn(BT, H, device=dev, generator=g).to(bf), dx=torch.empty_like(x)))
        w = (torch.rand(H, device=dev, generator=g) + 0.5).to(bf)
        dw = torch.empty_like(w)
        ws = torch.empty(L.lk_rmsnorm_bwd_workspace_bytes(BT, H), dtype=torch.uint8, device=dev)

        def mk_f(d):
            return lambda: _capi.check(L.lk_rmsnorm_fwd(d["x"].data_ptr(), w.data_ptr(), d["y"].data_ptr(),
                                                        d["rstd"].data_ptr(), BT, H, 1e-6, 0.0, 0, 1, st()))

        def mk_b(d):
            return lambda: _capi.check(L.lk_rmsnorm_bwd(d["dy"].data_ptr(), d["x"].data_ptr(), w.data_ptr(),
                                                        d["rstd"].data_ptr(), d["dx"].data_ptr(), dw.data_ptr(), BT,
                                                        H, 0.0, 0, 1, ws.data_ptr(), ws.numel(), st()))
        fb = 2 * BT * H * 2 + H * 2 + BT * 4
        bb = 3 * BT * H * 2 + H * 2 * 2 + BT * 4
        report("rmsnorm_fwd", fb, timed(mk_f(sets[0]), args.reps, flush),
               {"steady_ms": (sm_ := steady([mk_f(d) for d in sets], args.reps)),
                "steady_frac": fb / (sm_ / 1e3) / 1e9 / hbm})
        report("rmsnorm_bwd", bb, timed(mk_b(sets[0]), args.reps, flush),
               {"steady_ms": (sm_ := steady([mk_b(d) for d in sets], args.reps)),
                "steady_frac": bb / (sm_ / 1e3) / 1e9 / hbm})
        # diagnostic: the same backward without dgamma (no partial rows, no column-sum launch)
        nb = 3 * BT * H * 2 + H * 2 + BT * 4
        mk_nodw = lambda d: (lambda: _capi.check(L.lk_rmsnorm_bwd(  # noqa: E731
            d["dy"].data_ptr(), d["x"].data_ptr(), w.data_ptr(), d["rstd"].data_ptr(), d["dx"].data_ptr(), None, BT,
            H, 0.0, 0, 1, None, 0, st())))
        sm_ = steady([mk_nodw(d) for d in sets], args.reps)
        print(json.dumps({"kernel": "rmsnorm_bwd_no_dgamma (diagnostic)", "bytes": nb, "steady_ms": sm_,
                          "steady_frac": nb / (sm_ / 1e3) / 1e9 / hbm}), flush=True)
        del sets

    def both(name, nbytes, fns, extra=None):
        """cold-L2 single launch on the first buffer set + steady state over all sets"""
        sm_ = steady(fns, args.reps)
        line = {"steady_ms": sm_, "steady_frac": nbytes / (sm_ / 1e3) / 1e9 / hbm}
        if extra:
            line.update(extra)
        report(name, nbytes, timed(fns[0], args.reps, flush), line)

    # ---- LayerNorm (x: 8192 x 4096) ----
    if want("layernorm"):
        w = (torch.rand(H, device=dev, generator=g) + 0.5).to(bf)
        b = torch.randn(H, device=dev, generator=g).to(bf)
        dw, db = torch.empty_like(w), torch.empty_like(b)
        ws = torch.empty(L.lk_layernorm_bwd_workspace_bytes(BT, H), dtype=torch.uint8, device=dev)
        sets = []
        for _ in range(4):
            x = torch.randn(BT, H, device=dev, generator=g).to(bf)
            sets.append(dict(x=x, y=torch.empty_like(x), dy=torch.randn(BT, H, device=dev, generator=g).to(bf),
                             dx=torch.empty_like(x), mu=torch.empty(BT, device=dev), rs=torch.empty(BT, device=dev)))

        def ln_f(d):
            return lambda: _capi.check(L.lk_layernorm_fwd(d["x"].data_ptr(), w.data_ptr(), b.data_ptr(),
                                                          d["y"].data_ptr(), d["mu"].data_ptr(), d["rs"].data_ptr(),
                                                          BT, H, 1e-6, 1, st()))

        def ln_b(d):
            return lambda: _capi.check(L.lk_layernorm_bwd(d["dy"].data_ptr(), d["x"].data_ptr(), w.data_ptr(),
                                                          d["mu"].data_ptr(), d["rs"].data_ptr(), d["dx"].data_ptr(),
                                                          dw.data_ptr(), db.data_ptr(), BT, H, 1, ws.data_ptr(),
                                                          ws.numel(), st()))
        for d in sets:
            ln_f(d)()
        both("layernorm_fwd", 2 * BT * H * 2 + 2 * H * 2 + 2 * BT * 4, [ln_f(d) for d in sets])
        both("layernorm_bwd", 3 * BT * H * 2 + 3 * H * 2 + 2 * BT * 4, [ln_b(d) for d in sets])
        del sets

    # ---- RoPE (q: 4 x 2048 x 32 x 128, k: 4 x 2048 x 8 x 128; in place) ----
    if want("rope"):
        B, T = 4, 2048
        ang = torch.rand(1, T, D, device=dev, generator=g) * 6.28  # unit rotations: repeated in-place
        cos, sin = torch.cos(ang).to(bf), torch.sin(ang).to(bf)     # application stays bounded
        sets = [dict(q=torch.randn(B, T, NQ, D, device=dev, generator=g).to(bf),
                     k=torch.randn(B, T, NK, D, device=dev, generator=g).to(bf)) for _ in range(4)]
        nbytes = 2 * (sets[0]["q"].numel() + sets[0]["k"].numel()) * 2 + 2 * T * (D // 2) * 2
        for bwd in (0, 1):
            def rp(d, bwd=bwd):
                return lambda: _capi.check(L.lk_rope(d["q"].data_ptr(), d["k"].data_ptr(), cos.data_ptr(),
                                                     sin.data_ptr(), B, T, NQ, NK, D, 1, 1, 1, bwd, st()))
            both("rope_bwd" if bwd else "rope_fwd", nbytes, [rp(d) for d in sets])
        del sets

    # ---- SwiGLU / GeGLU (8192 x 14336) ----
    for kind in ("swiglu", "geglu"):
        if not want(kind):
            continue
        n = BT * I
        ffn, bfn = getattr(L, f"lk_{kind}_fwd"), getattr(L, f"lk_{kind}_bwd")
        sets = [dict(a=torch.randn(BT, I, device=dev, generator=g).to(bf),
                     b=torch.randn(BT, I, device=dev, generator=g).to(bf),
                     c=torch.empty(BT, I, device=dev, dtype=bf),
                     dc=(torch.randn(BT, I, device=dev, generator=g) * 1e-3).to(bf)) for _ in range(2)]

        def gf(d):
            return lambda: _capi.check(ffn(d["a"].data_ptr(), d["b"].data_ptr(), d["c"].data_ptr(), n, 1, st()))

        def gb(d):  # da/db overwrite a/b in place: the steady loop re-differentiates them
            return lambda: _capi.check(bfn(d["dc"].data_ptr(), d["a"].data_ptr(), d["b"].data_ptr(), n, 1, st()))
        both(f"{kind}_fwd", 3 * n * 2, [gf(d) for d in sets])
        both(f"{kind}_bwd", 5 * n * 2, [gb(d) for d in sets])
        del sets

    # ---- standalone cross entropy (8192 x 128256 bf16, in place) ----
    if want("cross_entropy"):
        rows = BT
        ws = torch.empty(256, dtype=torch.uint8, device=dev)
        ls = torch.empty((), device=dev)
        sets = [dict(x=torch.randn(rows, V, device=dev, generator=g).to(bf),
                     t=torch.randint(0, V, (rows,), device=dev, generator=g),
                     lr=torch.empty(rows, device=dev)) for _ in range(2)]

        def cef(d):
            return lambda: _capi.check(L.lk_cross_entropy_fwd(d["x"].data_ptr(), V, d["t"].data_ptr(), rows, V, 1,
                                                              -100, 0.0, 0.0, 0.0, 1, 1, d["lr"].data_ptr(),
                                                              ls.data_ptr(), None, None, ws.data_ptr(), ws.numel(),
                                                              st()))
        both("cross_entropy_fwd_bwd", 2 * rows * V * 2, [cef(d) for d in sets],
             {"note": "algorithmic bytes = 1 read + 1 write of the logits (the in-place minimum)"})
        del sets
    print(json.dumps({"summary": {o["kernel"]: {"cold": round(o["frac"], 3), "steady": round(o["steady_frac"], 3)}
                                  for o in out}}), flush=True)


if __name__ == "__main__":
    main()
