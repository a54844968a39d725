#!/bin/bash
# round-end style verification: full GPU suite, smoke, default bench, cfg4 + vocab bench, kernel bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
T=s4h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${T}_smoke.log
python bench.py 2>/dev/null | tail -1 > gpurun_out/prof/r01_bench.jsonl
python bench.py --config cfg4 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/prof/r01_bench_cfg4.jsonl
python bench.py --mode vocab --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/prof/r01_bench_vocab_n1.jsonl
python bench.py --impl reference 2>/dev/null | tail -1 > gpurun_out/prof/r01_bench_reference.jsonl
python bench_kernels.py --reps 30 > gpurun_out/prof/r01_kernels.jsonl 2>&1
for f in gpurun_out/prof/r01_bench*.jsonl; do echo "$f: $(cut -c1-300 $f)"; done
tail -1 gpurun_out/prof/r01_kernels.jsonl
