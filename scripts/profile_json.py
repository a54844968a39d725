"""Turn one ncu --set full capture of an FLCE step into profiles/<name>.json + .md (run here).

    python scripts/profile_json.py gpurun_out/X.ncu-rep profiles/r01_flce_step --bt 8192 --hidden 4096 --vocab 128256

The capture must hold exactly one FLCE step's GEMM and finalize launches in order
(chunk by chunk: logits GEMM, finalize, backward GEMM).  Per launch: duration, DRAM
bytes, tensor-pipe activity and -- for GEMM launches -- the algorithmic FLOP of that
launch (2*r*H*V logits, 4*r*H*V backward).  bench.py reads `dram_bytes_per_step` and
`gemm_dram_bytes_per_launch` from the JSON for its roofline `traffic` field.
"""

import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_active_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0, "%": 1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--bt", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=128256)
    ap.add_argument("--chunk", type=int, default=2048)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    name_i = hdr.index("Kernel Name")
    launches = []
    chunk_i = 0
    pending_logits = True
    for r in data:
        d = {"kernel": r[name_i][:80]}
        for k, lab in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                d[lab] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        if "gemm" in d["kernel"]:
            rows_c = min(a.chunk, a.bt - chunk_i * a.chunk)
            if pending_logits:
                d["role"] = f"logits chunk {chunk_i}"
                d["flop"] = 2.0 * rows_c * a.hidden * a.vocab
            else:
                d["role"] = f"backward chunk {chunk_i}"
                d["flop"] = 4.0 * rows_c * a.hidden * a.vocab
                chunk_i += 1
            pending_logits = not pending_logits
            d["tflops"] = d["flop"] / d["duration"] / 1e12
        else:
            d["role"] = f"finalize chunk {chunk_i}"
        d["dram_bytes"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        launches.append(d)
    gemm = [d for d in launches if "gemm" in d["kernel"]]
    out = {
        "source": a.rep,
        "shape": {"bt": a.bt, "hidden": a.hidden, "vocab": a.vocab, "chunk_rows": a.chunk},
        "launches": launches,
        "dram_bytes_per_step": sum(d["dram_bytes"] for d in gemm),
        "gemm_dram_bytes_per_launch": sum(d["dram_bytes"] for d in gemm) / max(1, len(gemm)),
        "gemm_flop_per_step": sum(d["flop"] for d in gemm),
        "gemm_ms_per_step_cold": sum(d["duration"] for d in gemm) * 1e3,
        "note": "ncu replay: cold cache, serialised launches; compare shares, not absolute step time",
    }
    with open(a.out + ".json", "w") as f:
        json.dump(out, f, indent=1)
    lines = [f"# FLCE step, ncu --set full (`{a.rep}`)\n", out["note"] + "\n",
             "| launch | role | ms | TFLOP/s | tensor active % | DRAM GB | SM GHz |", "|---|---|---|---|---|---|---|"]
    for i, d in enumerate(launches):
        lines.append(f"| {i} `{d['kernel'][:40]}` | {d['role']} | {d['duration']*1e3:.3f} | "
                     f"{d.get('tflops', 0):.0f} | {d.get('tensor_active_pct', 0):.1f} | {d['dram_bytes']/1e9:.3f} | "
                     f"{d.get('sm_clock', 0)/1e9:.2f} |")
    lines.append(f"\nGEMM DRAM bytes per step: {out['dram_bytes_per_step']/1e9:.2f} GB; "
                 f"GEMM time per step (cold): {out['gemm_ms_per_step_cold']:.2f} ms; "
                 f"GEMM FLOP per step {out['gemm_flop_per_step']:.3e}")
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
