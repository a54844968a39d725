#!/bin/bash
# round-2 final validation: full -m gpu suite, smoke, default bench line (driver invocation), kernel bench
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2an_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r2an_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2an_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2an_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2an_smoke.log
timeout 900 python bench.py > gpurun_out/r2an_bench.jsonl 2> gpurun_out/r2an_bench.err
timeout 600 python bench_kernels.py > gpurun_out/r2an_kernels.jsonl 2>&1
grep -E "passed|failed|rc=" gpurun_out/r2an_gputests.log | tail -3; tail -2 gpurun_out/r2an_smoke.log
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2an_bench.jsonl").read().strip().splitlines()[-1])
print(round(d["value"]), round(d["e2e"]["value"]), round(d["roofline"]["frac"], 3), d["clocks"], d["gpu_launches"])
PY
tail -1 gpurun_out/r2an_kernels.jsonl
