#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider -k "large_vocab or rmsnorm or rope" > gpurun_out/gpu_tests2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests2.log
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/kernels.log 2>&1; echo "rc=$?" >> gpurun_out/kernels.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python scripts/profile_flce.py --steps 2 > gpurun_out/ncu_launch.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 4 -c 2 -o gpurun_out/r01_gemm python scripts/profile_flce.py --steps 2 > gpurun_out/ncu_gemm.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:ce_rows -s 2 -c 1 -o gpurun_out/r01_finalize python scripts/profile_flce.py --steps 1 > gpurun_out/ncu_fin.log 2>&1
timeout -s KILL 400 ncu --set full --clock-control none -k "regex:rmsnorm|rope|glu" -c 12 -o gpurun_out/r01_rowops python bench_kernels.py --reps 1 --only rmsnorm,rope,swiglu,geglu > gpurun_out/ncu_rowops.log 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/gpu_tests2.log gpurun_out/kernels.log gpurun_out/bench.log gpurun_out/ncu_gemm.log
ls -la gpurun_out
