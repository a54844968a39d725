#!/bin/bash
# full default bench line (incl. fp32 cfg2 variant + CPU baselines), reference arm, --gpus 2 on the
# one-GPU lease (LK_BENCH_SHARE_GPU: a path check, not a bench value), BenchRecord f32 + bf16 rows
cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py > gpurun_out/r2k_bench_n1.jsonl 2> gpurun_out/r2k_bench_n1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2k_bench_ref.jsonl 2> gpurun_out/r2k_bench_ref.err
LK_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/r2k_bench_share2.jsonl 2> gpurun_out/r2k_bench_share2.err
echo "share2 rc=$?" >> gpurun_out/r2k_bench_share2.err
timeout 900 python -m paper_2410_10989_b200.benchrecord --dtype f32 --out gpurun_out/r2k_benchrecord_gpu_f32.csv > /dev/null 2> gpurun_out/r2k_br.err
timeout 900 python -m paper_2410_10989_b200.benchrecord --dtype bf16 --out gpurun_out/r2k_benchrecord_gpu_bf16.csv > /dev/null 2>> gpurun_out/r2k_br.err
head -c 600 gpurun_out/r2k_bench_n1.jsonl; echo; tail -c 300 gpurun_out/r2k_bench_ref.jsonl; echo; head -c 400 gpurun_out/r2k_bench_share2.jsonl; tail -2 gpurun_out/r2k_bench_share2.err; wc -l gpurun_out/r2k_benchrecord_gpu_*.csv
