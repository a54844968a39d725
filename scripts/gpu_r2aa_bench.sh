#!/bin/bash
# round-2 bench lines after the kernel and bench changes: default (driver invocation), cfg4, vocab N=1, cfg5 N=1
cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py > gpurun_out/r2aa_bench_default.jsonl 2> gpurun_out/r2aa_bench_default.err
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2aa_bench_cfg4.jsonl 2>&1
timeout 600 python bench.py --mode vocab --steps 20 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/r2aa_bench_vocab_n1.jsonl 2>&1
timeout 600 python bench.py --config cfg5 --steps 4 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/r2aa_bench_cfg5_n1.jsonl 2>&1
for f in default cfg4 vocab_n1 cfg5_n1; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r2aa_bench_{f}.jsonl").read().strip().splitlines()[-1])
    print(f, round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms", round(d["ms_per_step"], 2), "frac", round(d["roofline"]["frac"], 3), d["clocks"])
except Exception as e:
    print(f, "ERR", e)
PY
done
