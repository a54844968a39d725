#!/bin/bash
# Round-1 session-2 GPU pass: build, parity tests, bench, kernel bench, ncu launch list + full captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/s2a_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s2a_build_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s2a_build_smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/s2a_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2a_gpu_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/s2a_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s2a_bench.log
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s2a_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/s2a_bench_ref.log
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/s2a_kernels.log 2>&1; echo "kernels rc=$?" >> gpurun_out/s2a_kernels.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2a_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/s2a_ncu_launch.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 6 -c 3 -o gpurun_out/s2a_gemm python scripts/profile_flce.py --steps 2 > gpurun_out/s2a_ncu_gemm.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:'ce_|rmsnorm|norm|rope|glu' -c 12 -o gpurun_out/s2a_rowops python bench_kernels.py --reps 1 > gpurun_out/s2a_ncu_rowops.log 2>&1
tail -3 gpurun_out/s2a_build_smoke.log gpurun_out/s2a_gpu_tests.log gpurun_out/s2a_bench.log gpurun_out/s2a_bench_ref.log gpurun_out/s2a_kernels.log
