#!/bin/bash
# one-step FLCE profile + launch list, summarised on the box (ncu-rep files are too big to return)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
T=s3c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none -k regex:'gemm|ce_ring' -s 12 -c 12 -o /tmp/${T}_flce_step python scripts/profile_flce.py --steps 2 > gpurun_out/${T}_ncu_flce.log 2>&1
python scripts/profile_json.py /tmp/${T}_flce_step.ncu-rep gpurun_out/prof/r01_flce_step > /dev/null 2>&1
python scripts/ncu_summary.py report /tmp/${T}_flce_step.ncu-rep > gpurun_out/prof/r01_flce_step_full.md 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/r01_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/prof/r01_bench.jsonl 2>&1
timeout -s KILL 300 python bench.py --impl reference > gpurun_out/prof/r01_bench_reference.jsonl 2>&1
timeout -s KILL 300 python bench.py --config cfg4 --steps 20 --no-cpu-baseline > gpurun_out/prof/r01_bench_cfg4.jsonl 2>&1
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/prof/r01_kernels.jsonl 2>&1
cat gpurun_out/prof/r01_flce_step.md
