"""ncu DRAM traffic of the FLCE GEMM launches, per local problem shape -> profiles/r02_traffic.json.

Run on the GPU box (one GPU, never under torchrun):

    python scripts/traffic_capture.py            # every shape bench.py can run locally
    python scripts/traffic_capture.py --inner 8192 4096 128256 0   # (internal) one profiled step

For each shape, ncu (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none --profile-from-start off`) records exactly one FLCE fwd+bwd step after
warm-up (cudaProfilerStart/Stop around it).  bench.py's roofline `traffic` reads
`gemm_dram_bytes_per_launch` for the shape it runs (key "bt{BT}_h{H}_v{V}_cap{softcap}").
"""

import argparse
import csv
import io
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

SHAPES = [  # (bt per GPU, H, V, softcap, smoothing, ignored rows skipped)
    (8192, 4096, 128256, 0.0, 0.0, 1),    # cfg2 (one GPU: the kept-row path)
    (65536, 4096, 128256, 0.0, 0.0, 1),   # cfg5 at N=1
    (8192, 3584, 256000, 30.0, 0.1, 1),   # cfg4
    (8192, 4096, 128256, 0.0, 0.0, 0),    # token-sharded ranks (no host read, all rows): cfg2 weak
    (16384, 4096, 128256, 0.0, 0.0, 0),   # and cfg5 at N=8 / 4 / 2
    (32768, 4096, 128256, 0.0, 0.0, 0),
]
METRICS = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "second": 1.0}


def key(bt, h, v, softcap, skip=0):
    return f"bt{bt}_h{h}_v{v}_cap{float(softcap or 0.0):g}" + ("_kept" if skip else "")


def inner(bt, h, v, softcap, smoothing, skip):
    import torch

    from paper_2410_10989_b200.fused_linear_cross_entropy import fused_linear_cross_entropy_forward as f

    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.rand(bt, h, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(v, h, device="cuda", generator=g) * 2 - 1) / 64.0).to(torch.bfloat16)
    t = torch.randint(0, v, (bt,), device="cuda", generator=g)
    t[torch.rand(bt, device="cuda", generator=g) < 0.1] = -100
    kw = dict(softcap=softcap or None, label_smoothing=smoothing, compute_grad_input=True, compute_grad_weight=True,
              skip_ignored_rows=bool(skip))
    for _ in range(2):
        f(x, w, t, **kw)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    f(x, w, t, **kw)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


def capture(shape, outdir, parse_only=False):
    bt, h, v, cap, ls, skip = shape
    log = outdir / f"traffic_{key(bt, h, v, cap, skip)}.csv"
    cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--profile-from-start", "off", "--csv",
           "--log-file", str(log), sys.executable, __file__, "--inner", str(bt), str(h), str(v), str(cap), str(ls),
           str(skip)]
    if not parse_only:
        subprocess.run(cmd, cwd=ROOT, check=True)
    rows = list(csv.reader(io.StringIO(log.read_text())))
    hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[hdr_i]
    per = {}
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        lid = d["ID"]
        val = float(d["Metric Value"].replace(",", "")) * SCALE.get(d.get("Metric Unit", ""), 1.0)
        e = per.setdefault(lid, {"kernel": d["Kernel Name"][:90]})
        e[d["Metric Name"]] = val
    launches = list(per.values())
    gemm = [e for e in launches if "gemm" in e["kernel"]]
    dram = lambda e: e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)  # noqa: E731
    return {
        "shape": {"bt": bt, "hidden": h, "vocab": v, "softcap": cap, "label_smoothing": ls,
                  "ignored_rows_skipped": bool(skip)},
        "n_launches": len(launches), "n_gemm_launches": len(gemm),
        "gemm_dram_bytes_per_launch": sum(map(dram, gemm)) / max(1, len(gemm)),
        "dram_bytes_per_step": sum(map(dram, launches)),
        "gemm_dram_bytes_per_step": sum(map(dram, gemm)),
        "gemm_ms_per_step_cold": 1e3 * sum(e.get("gpu__time_duration.sum", 0.0) for e in gemm),
        "step_ms_cold": 1e3 * sum(e.get("gpu__time_duration.sum", 0.0) for e in launches),
        "source": f"ncu --metrics {METRICS} --clock-control none, one step after warm-up ({log.name})",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--inner", nargs=6, default=None)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_traffic.json"))
    ap.add_argument("--logdir", default=str(ROOT / "gpurun_out"))
    ap.add_argument("--parse-only", action="store_true", help="rebuild --out from the CSVs already in --logdir")
    a = ap.parse_args()
    if a.inner:
        bt, h, v = (int(s) for s in a.inner[:3])
        inner(bt, h, v, float(a.inner[3]), float(a.inner[4]), int(a.inner[5]))
        return
    outdir = Path(a.logdir)
    outdir.mkdir(parents=True, exist_ok=True)
    res = {}
    for shape in SHAPES:
        k = key(*shape[:4], shape[5])
        try:
            res[k] = capture(shape, outdir, a.parse_only)
        except Exception as e:  # keep the other shapes
            res[k] = {"error": repr(e)[:300]}
        print(k, json.dumps(res[k])[:300], flush=True)
    Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
