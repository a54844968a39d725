#!/bin/bash
# run-to-run spread of the headline bench line on one box (5 default runs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
for i in 1 2 3 4 5; do
  python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'run': $i, 'value': round(d['value']), 'e2e': round(d['e2e']['value']), 'ms_per_step': round(d['ms_per_step'],3), 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons'], 'gemm_tflops': round(d['roofline']['achieved'],1)}))"
done | tee gpurun_out/prof/r01_bench_spread.jsonl
