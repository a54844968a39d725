#!/bin/bash
# round-2 bench: N=1 cfg2 default line, cfg4, cfg5 (N=1), the --gpus 2 self-launch path on one
# GPU (LK_BENCH_SHARE_GPU, not a bench value), and per-shape ncu DRAM traffic.
cd "$GRAFT_REPO_ROOT"
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_n1.jsonl 2> gpurun_out/r2_bench_n1.err
python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg4.jsonl 2>&1
python bench.py --config cfg5 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_n1.jsonl 2>&1
LK_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-variants > gpurun_out/r2_bench_share2.jsonl 2>&1
echo "share2 rc=$?" >> gpurun_out/r2_bench_share2.jsonl
timeout 1200 python scripts/traffic_capture.py > gpurun_out/r2_traffic.log 2>&1
cp profiles/r02_traffic.json gpurun_out/ 2>/dev/null
tail -c 600 gpurun_out/r2_bench_n1.jsonl
