#!/bin/bash
# ncu --set full of one logits GEMM (gemm2_kernel, FLCE chunk 0) and one backward GEMM launch:
# raw metrics + warp-stall summary for the next round's GEMM work (profiles/r01_gemm_stalls.md)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
T=s4k
timeout -s KILL 900 ncu --set full --clock-control none -k regex:gemm2 -s 8 -c 2 -o /tmp/${T}_gemm python scripts/profile_flce.py --steps 2 > gpurun_out/${T}_ncu.log 2>&1
ncu -i /tmp/${T}_gemm.ncu-rep --page raw --csv > /tmp/${T}_raw.csv 2>/dev/null
python - <<'PY' > gpurun_out/prof/r01_gemm_stalls.md
import csv, re
rows = list(csv.reader(open("/tmp/s4k_raw.csv")))
hdr, data = rows[0], rows[2:]
print("# tcgen05 GEMM warp-state breakdown (ncu --set full, FLCE step launches 8-9: logits + backward)\n")
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]
for n, r in enumerate(data):
    d = dict(zip(hdr, r))
    print(f"## launch {n}\n\n| metric | value |\n|---|---|")
    for k in keys:
        print(f"| `{k}` | {d.get(k, '')} |")
    st = []
    for k in hdr:
        m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active\.ratio$", k)
        if m:
            try: st.append((float(d[k]), m.group(1)))
            except ValueError: pass
    print("\n| stall reason (warps per issue) | value |\n|---|---|")
    for v, name in sorted(st, reverse=True)[:10]:
        print(f"| {name} | {v:.3f} |")
    print()
PY
cat gpurun_out/prof/r01_gemm_stalls.md | head -60
