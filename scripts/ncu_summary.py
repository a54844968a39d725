"""Summarise ncu output for profiles/ (run here, on the CPU box, after gpurun).

    python scripts/ncu_summary.py launches gpurun_out/r01_launches.csv > profiles/r01_launches.md
    python scripts/ncu_summary.py report gpurun_out/r01_gemm.ncu-rep [--flops F1,F2,...] > profiles/r01_gemm.md
"""

import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster x"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return f * scale


def to_ms(v, unit):
    f = float(v.replace(",", ""))
    return f * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}.get(unit, 1.0)


def report(path, flops=None):
    rows = ncu_csv(["-i", path, "--page", "raw"])
    hdr, units, data = rows[0], rows[1], rows[2:]
    print(f"# ncu --set full summary: `{path}`\n")
    name_i = hdr.index("Kernel Name")
    for n, r in enumerate(data):
        print(f"## launch {n}: `{r[name_i][:90]}`\n")
        print("| metric | value |\n|---|---|")
        dur_ms = None
        traffic = 0.0
        for key, label in METRICS:
            if key not in hdr:
                continue
            i = hdr.index(key)
            val, unit = r[i], units[i]
            if key == "gpu__time_duration.sum":
                dur_ms = to_ms(val, unit)
            if key.startswith("dram__bytes"):
                traffic += to_bytes(val, unit)
            print(f"| {label} (`{key}`) | {val} {unit} |")
        print(f"| DRAM traffic (read + write) | {traffic / 1e9:.3f} GB |")
        if flops and n < len(flops) and dur_ms:
            tf = flops[n] / (dur_ms / 1e3) / 1e12
            print(f"| algorithmic FLOP | {flops[n]:.4g} |\n| achieved (cold, serialised, under ncu) | {tf:.0f} TFLOP/s |")
        print()


def launches(path):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[i0 + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("void ", "")[:70]
            tot[name] += to_ms(r[vi], r[ui])
            cnt[name] += 1
    s = sum(tot.values())
    print(f"# launch list: `{path}` (ncu, cold cache, serialised: compare shares)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.3f} | {v / s * 100:.1f}% |")
    print(f"| **all** | {sum(cnt.values())} | {s:.3f} | 100% |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        fl = None
        if "--flops" in sys.argv:
            fl = [float(x) for x in sys.argv[sys.argv.index("--flops") + 1].split(",")]
        report(sys.argv[2], fl)
