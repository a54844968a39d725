"""Bench results in the reference's BenchRecord CSV schema.

`rowfuse report results.csv` (rowfuse/cli.py:275-289) merges "fused" / "reference" rows
of this schema into a speedup / memory-ratio table (rowfuse/bench.py:375-404).  This
module times the sm_100a kernels at the reference's default bench shapes
(rowfuse/bench.py:49-62) and writes them as variant "fused" records, so a reference user
can drop the GPU numbers next to their CPU runs.  The timing protocol is the reference's:
3 warm-ups, then `repeats` timed forward+backward calls, median and the [0.2, 0.8]
quantiles (rowfuse/bench.py:46-48, 315-324) -- here with CUDA events on the launching
stream; peak_bytes is the allocator's peak above the inputs during one call.

    python -m paper_2410_10989_b200.benchrecord --out gpu_results.csv [--ops rmsnorm,linear_ce]
"""

from __future__ import annotations

import argparse
import csv
import statistics
from dataclasses import dataclass

import torch

FIELDS = ("op", "variant", "rows", "cols", "hidden", "dtype", "repeats", "workers", "median_s", "q20_s", "q80_s",
          "peak_bytes")  # rowfuse/bench.py:84-97 (column order is the schema)
HIDDEN_SWEEP = (4096, 8192, 12288, 16384)  # rowfuse/bench.py:43-44
VOCAB_SWEEP = (40960, 81920, 122880, 163840)
OPS = ("rmsnorm", "layernorm", "rope", "swiglu", "geglu", "cross_entropy", "linear_ce")
DTYPES = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


class SchemaMismatch(ValueError):
    """Mirrors rowfuse.bench.SchemaMismatch."""


@dataclass(frozen=True)
class BenchRecord:  # rowfuse/bench.py:100-130
    op: str
    variant: str
    rows: int
    cols: int
    hidden: int
    dtype: str
    repeats: int
    workers: int
    median_s: float
    q20_s: float
    q80_s: float
    peak_bytes: int

    def to_row(self) -> list[str]:
        return [self.op, self.variant, str(self.rows), str(self.cols), str(self.hidden), self.dtype, str(self.repeats),
                str(self.workers), repr(self.median_s), repr(self.q20_s), repr(self.q80_s), str(self.peak_bytes)]


def write_records(path, records) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(FIELDS)
        for r in records:
            w.writerow(r.to_row())


def read_records(path) -> list[BenchRecord]:
    """Same validation as rowfuse/bench.py:141-159."""
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header != list(FIELDS):
            raise SchemaMismatch(f"expected columns {FIELDS}, found {header}")
        out = []
        for row in reader:
            if len(row) != len(FIELDS):
                raise SchemaMismatch(f"row has {len(row)} fields, expected {len(FIELDS)}")
            kw = dict(zip(FIELDS, row))
            try:
                for k in ("rows", "cols", "hidden", "repeats", "workers", "peak_bytes"):
                    kw[k] = int(kw[k])
                for k in ("median_s", "q20_s", "q80_s"):
                    kw[k] = float(kw[k])
            except ValueError as exc:
                raise SchemaMismatch(f"unparseable row {row}: {exc}") from None
            out.append(BenchRecord(**kw))
        return out


def default_shapes(op: str):
    """(rows, cols, hidden) of rowfuse/bench.py:52-62."""
    if op in ("rmsnorm", "layernorm", "rope"):
        return tuple((256, c, 0) for c in HIDDEN_SWEEP)
    if op in ("swiglu", "geglu"):
        return tuple((r, 512, 0) for r in HIDDEN_SWEEP)
    if op == "cross_entropy":
        return tuple((512, v, 0) for v in VOCAB_SWEEP)
    if op == "linear_ce":
        return tuple((128, v, 256) for v in VOCAB_SWEEP)
    raise ValueError(f"unknown op {op!r}")


def _case(op, rows, cols, hidden, dtype, dev):
    """Returns (inputs kept alive, fn running forward + backward once)."""
    import paper_2410_10989_b200 as lk

    g = torch.Generator(device=dev).manual_seed(0)
    r = lambda *s: (torch.rand(*s, device=dev, generator=g) * 2 - 1).to(dtype)  # noqa: E731
    if op in ("rmsnorm", "layernorm"):
        x, w, b, dy = r(rows, cols), r(cols).abs() + 0.5, r(cols), r(rows, cols)

        def fn():
            xr, wr = x.clone().requires_grad_(True), w.clone().requires_grad_(True)
            if op == "rmsnorm":
                y = lk.liger_rms_norm(xr, wr, 1e-6, 0.0, "llama", False)
            else:
                y = lk.liger_layer_norm(xr, wr, b.clone().requires_grad_(True), 1e-6)
            y.backward(dy)
        return (x, w, b, dy), fn
    if op == "rope":  # rowfuse rotates q and k of equal shape, one head of width `cols`
        q, k = r(1, rows, 1, cols), r(1, rows, 1, cols)
        ang = torch.arange(rows, device=dev)[:, None] * (1e4 ** (-torch.arange(0, cols, 2, device=dev) / cols))[None]
        cos = torch.cat([ang, ang], -1).cos()[None].to(dtype)
        sin = torch.cat([ang, ang], -1).sin()[None].to(dtype)

        def fn():
            qq = q.clone().transpose(1, 2).requires_grad_(True)
            kk = k.clone().transpose(1, 2).requires_grad_(True)
            qo, ko = lk.liger_rotary_pos_emb(qq, kk, cos, sin)
            (qo.float().sum() + ko.float().sum()).backward()
        return (q, k, cos, sin), fn
    if op in ("swiglu", "geglu"):
        a, b2, dc = r(rows, cols), r(rows, cols), r(rows, cols)
        f = lk.LigerSiLUMulFunction if op == "swiglu" else lk.LigerGELUMulFunction

        def fn():
            f.apply(a.clone().requires_grad_(True), b2.clone().requires_grad_(True)).backward(dc)
        return (a, b2, dc), fn
    if op == "cross_entropy":
        z = r(rows, cols) * 4
        t = torch.randint(0, cols, (rows,), device=dev, generator=g)

        def fn():
            lk.LigerCrossEntropyLoss()(z.clone().requires_grad_(True), t).backward()
        return (z, t), fn
    if op == "linear_ce":
        x, w = r(rows, hidden), r(cols, hidden) / hidden ** 0.5
        t = torch.randint(0, cols, (rows,), device=dev, generator=g)

        def fn():
            lk.LigerFusedLinearCrossEntropyLoss()(w.clone().requires_grad_(True), x.clone().requires_grad_(True),
                                                  t).backward()
        return (x, w, t), fn
    raise ValueError(op)


def bench_op(op, rows, cols, hidden, dtype_name="bf16", repeats=10, device="cuda") -> BenchRecord:
    dev = torch.device(device)
    dtype = DTYPES[dtype_name]
    keep, fn = _case(op, rows, cols, hidden, dtype, dev)
    for _ in range(3):
        fn()
    torch.cuda.synchronize(dev)
    base = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    times = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize(dev)
        times.append(e0.elapsed_time(e1) / 1e3)
    peak = torch.cuda.max_memory_allocated(dev) - base
    qs = statistics.quantiles(times, n=5) if len(times) >= 2 else [times[0]] * 4
    del keep
    return BenchRecord(op, "fused", rows, cols, hidden, dtype_name, repeats, 0, statistics.median(times), qs[0], qs[3],
                       int(peak))


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--out", required=True)
    ap.add_argument("--ops", default=",".join(OPS))
    ap.add_argument("--dtype", default="bf16", choices=sorted(DTYPES))
    ap.add_argument("--repeats", type=int, default=10)
    a = ap.parse_args(argv)
    recs = [bench_op(op, r, c, h, a.dtype, a.repeats) for op in a.ops.split(",") for r, c, h in default_shapes(op)]
    write_records(a.out, recs)
    for rec in recs:
        print(",".join(rec.to_row()))


if __name__ == "__main__":
    main()
