"""Same-box comparison on B200: this library vs the upstream Liger-Kernel (liger_kernel 0.8.0,
Triton, installed in the image) vs torch eager, on the north-star workloads.

Not part of the product or the tests: a measurement script.  Each op runs forward + backward
through its public module/function; timing is CUDA events around the call (median of
`--reps` after 3 warm-ups), inputs resident in HBM; `graph_ms` (small ops) is the GPU time
per call with 10 calls captured in one CUDA graph (host launch cost out of the loop); peak memory = allocator peak above
the inputs during one call.

    python scripts/compare_liger.py [--reps 10] [--only flce,ce,rmsnorm,rope,swiglu,layernorm]
"""

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed.tensor  # noqa: E402,F401  (liger_kernel checks isinstance(x, DTensor))
import torch.nn.functional as F  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), (torch.cuda.max_memory_allocated() - base) / 2**20


def graph_timed(fn, calls=10, replays=5):
    """GPU time per call with the host out of the loop: `calls` calls captured in one CUDA graph,
    replayed; None when the implementation cannot be captured (a host sync inside)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            for _ in range(calls):
                fn()
    except Exception:
        torch.cuda.synchronize()
        return None
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(replays):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / calls)
    del g
    return statistics.median(ts)


def run(name, impls, reps, out, graph=False):
    for impl, fn in impls:
        try:
            ms, mb = timed(fn, reps)
            rec = {"op": name, "impl": impl, "ms": round(ms, 4), "peak_mib": round(mb, 1)}
            if graph:
                gms = graph_timed(fn)
                rec["graph_ms"] = None if gms is None else round(gms, 4)
        except Exception as exc:  # e.g. an upstream kernel that does not run on sm_100
            rec = {"op": name, "impl": impl, "error": f"{type(exc).__name__}: {str(exc)[:160]}"}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="flce,flce_gemma,ce,rmsnorm,layernorm,rope,swiglu")
    a = ap.parse_args()
    want = set(a.only.split(","))
    import liger_kernel.transformers as lkt
    from liger_kernel.transformers.rope import liger_rotary_pos_emb as up_rope

    import paper_2410_10989_b200 as lk

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    bf = torch.bfloat16
    out = []

    def flce_case(name, bt, h, v, **kw):
        x = (torch.rand(bt, h, device=dev, generator=g) * 2 - 1).to(bf)
        w = ((torch.rand(v, h, device=dev, generator=g) * 2 - 1) / h ** 0.5).to(bf)
        t = torch.randint(0, v, (bt,), device=dev, generator=g)
        t[::10] = -100
        ours, up = lk.LigerFusedLinearCrossEntropyLoss(**kw), lkt.LigerFusedLinearCrossEntropyLoss(**kw)

        def mk(mod):
            def f():
                xx, ww = x.detach().requires_grad_(True), w.detach().requires_grad_(True)
                mod(ww, xx, t).backward()
            return f

        def eager():
            xx, ww = x.detach().requires_grad_(True), w.detach().requires_grad_(True)
            z = (xx @ ww.t()).float()
            if kw.get("softcap"):
                z = kw["softcap"] * torch.tanh(z / kw["softcap"])
            F.cross_entropy(z, t, ignore_index=-100, label_smoothing=kw.get("label_smoothing", 0.0)).backward()

        run(name, [("b200", mk(ours)), ("liger_triton", mk(up)), ("torch_eager", eager)], a.reps, out)

    if "flce" in want:
        flce_case("flce cfg2 (8192x4096x128256)", 8192, 4096, 128256)
    if "flce_gemma" in want:
        flce_case("flce cfg4 (8192x3584x256000, softcap 30, ls 0.1)", 8192, 3584, 256000, softcap=30.0,
                  label_smoothing=0.1)
    if "ce" in want:
        z = (torch.randn(8192, 128256, device=dev, generator=g) * 3).to(bf)
        t = torch.randint(0, 128256, (8192,), device=dev, generator=g)

        def mk(mod):
            def f():
                zz = z.detach().clone().requires_grad_(True)
                mod(zz, t).backward()
            return f
        # the clone (2.1 GB copy) is inside every impl's timed region alike
        run("cross_entropy 8192x128256 (+clone)", [("b200", mk(lk.LigerCrossEntropyLoss())),
                                                   ("liger_triton", mk(lkt.LigerCrossEntropyLoss())),
                                                   ("torch_eager", mk(lambda zz, tt: F.cross_entropy(zz.float(), tt)))],
            a.reps, out, graph=True)
        del z
    x = (torch.rand(8192, 4096, device=dev, generator=g) * 2 - 1).to(bf)
    dy = (torch.rand(8192, 4096, device=dev, generator=g) * 2 - 1).to(bf)
    if "rmsnorm" in want:
        ours, up = lk.LigerRMSNorm(4096).to(dev, bf), lkt.LigerRMSNorm(4096).to(dev, bf)

        def mk(mod):
            def f():
                xx = x.detach().requires_grad_(True)
                mod(xx).backward(dy)
            return f

        def eager():
            xx = x.detach().requires_grad_(True)
            xf = xx.float()
            (ours.weight * (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-6)).to(bf)).backward(dy)
        run("rmsnorm 8192x4096", [("b200", mk(ours)), ("liger_triton", mk(up)), ("torch_eager", eager)], a.reps, out,
            graph=True)
    if "layernorm" in want:
        ours, up = lk.LigerLayerNorm(4096).to(dev, bf), lkt.LigerLayerNorm(4096).to(dev, bf)
        ref = torch.nn.LayerNorm(4096).to(dev, bf)

        def mk(mod):
            def f():
                xx = x.detach().requires_grad_(True)
                mod(xx).backward(dy)
            return f
        run("layernorm 8192x4096", [("b200", mk(ours)), ("liger_triton", mk(up)), ("torch_eager", mk(ref))], a.reps,
            out, graph=True)
    if "rope" in want:
        b, t_, nq, nk, d = 4, 2048, 32, 8, 128
        q0 = torch.randn(b, t_, nq, d, device=dev, generator=g).to(bf)
        k0 = torch.randn(b, t_, nk, d, device=dev, generator=g).to(bf)
        ang = torch.arange(t_, device=dev)[:, None] * (5e5 ** (-torch.arange(0, d, 2, device=dev) / d))[None]
        emb = torch.cat([ang, ang], -1)[None]
        cos, sin = emb.cos().to(bf), emb.sin().to(bf)

        def mk(fn):
            def f():
                q = q0.detach().clone().transpose(1, 2).requires_grad_(True)
                k = k0.detach().clone().transpose(1, 2).requires_grad_(True)
                qo, ko = fn(q, k, cos, sin)
                torch.autograd.backward([qo, ko], [torch.ones_like(qo), torch.ones_like(ko)])
            return f

        def rot(x_, c, s):
            h = x_.shape[-1] // 2
            return x_ * c + torch.cat([-x_[..., h:], x_[..., :h]], -1) * s

        def eager_fn(q, k, c, s):
            return rot(q, c[:, None], s[:, None]), rot(k, c[:, None], s[:, None])
        run("rope 4x2048, 32q/8kv heads x128 (+clones)", [("b200", mk(lk.liger_rotary_pos_emb)),
                                                         ("liger_triton", mk(up_rope)),
                                                         ("torch_eager", mk(eager_fn))], a.reps, out, graph=True)
    if "swiglu" in want:
        a_ = torch.randn(8192, 14336, device=dev, generator=g).to(bf)
        b_ = torch.randn(8192, 14336, device=dev, generator=g).to(bf)
        dc = torch.randn(8192, 14336, device=dev, generator=g).to(bf)
        from liger_kernel.ops.swiglu import LigerSiLUMulFunction as UpSiLU

        def mk(fn):
            def f():
                aa, bb = a_.detach().clone().requires_grad_(True), b_.detach().clone().requires_grad_(True)
                fn(aa, bb).backward(dc)
            return f
        run("swiglu 8192x14336 (+clones)", [("b200", mk(lk.LigerSiLUMulFunction.apply)),
                                            ("liger_triton", mk(UpSiLU.apply)),
                                            ("torch_eager", mk(lambda aa, bb: F.silu(aa) * bb))], a.reps, out,
            graph=True)
    print(json.dumps({"summary": out}))


if __name__ == "__main__":
    main()
