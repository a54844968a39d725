#!/bin/bash
# fp32 split operands addressed by piece (no duplicated term copies): fp32 parity tests, converge,
# fp32 timings (cfg1, cfg2 shape), BenchRecord linear_ce f32 rows
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_parity_headline.py tests/test_gpu_flce.py tests/test_converge.py tests/test_gpu_gemm.py tests/test_gpu_distributed.py -m gpu -q -p no:cacheprovider > gpurun_out/r2ad_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2ad_tests.log
timeout 600 python scripts/probe_tc_accum.py 2>&1 | grep flce_fp32 > gpurun_out/r2ad_probe.jsonl
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2ad_bench.jsonl 2> gpurun_out/r2ad_bench.err
timeout 600 python -m paper_2410_10989_b200.benchrecord --dtype f32 --ops linear_ce --out gpurun_out/r2ad_br_f32.csv > /dev/null 2>&1
tail -3 gpurun_out/r2ad_tests.log; cat gpurun_out/r2ad_probe.jsonl; cat gpurun_out/r2ad_br_f32.csv
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2ad_bench.jsonl").read().strip().splitlines()[-1])
print(d["variants"]["fp32_cfg2"]); print(d["cpu_baseline"]["cfg1"]["gpu_fp32"])
PY
