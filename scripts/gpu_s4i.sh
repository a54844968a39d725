#!/bin/bash
# refresh the one-step FLCE ncu capture (12 launches) and the launch list of bench.py
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
T=s4i
timeout -s KILL 900 ncu --set full --clock-control none -k regex:'gemm|ce_ring' -s 12 -c 12 -o /tmp/${T}_flce_step python scripts/profile_flce.py --steps 2 > gpurun_out/${T}_ncu_flce.log 2>&1
python scripts/profile_json.py /tmp/${T}_flce_step.ncu-rep gpurun_out/prof/r01_flce_step > /dev/null 2>&1
python scripts/ncu_summary.py report /tmp/${T}_flce_step.ncu-rep > gpurun_out/prof/r01_flce_step_full.md 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/r01_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/prof/r01_launches.csv > gpurun_out/prof/r01_launches.md 2>&1
ls -la gpurun_out/prof; head -20 gpurun_out/prof/r01_flce_step.md
