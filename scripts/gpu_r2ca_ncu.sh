#!/bin/bash
# ncu evidence for the round-2 final path (kept rows, 3-chunk plan): per-shape DRAM traffic for
# roofline.traffic, the launch list of the bench command, and a --set full capture of one
# logits GEMM + one backward GEMM + the finalize of the kept-row cfg2 step.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2ca
timeout 1500 python scripts/traffic_capture.py --logdir gpurun_out > ${O}_traffic.log 2>&1
tail -8 ${O}_traffic.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-variants > ${O}_launches_bench.log 2>&1
tail -c 300 ${O}_launches_bench.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"gemm2_kernel|ce_ring" -s 12 -c 3 \
  -o ${O}_step python scripts/skip_chunk_probe.py 1 1:0 > ${O}_full.log 2>&1
tail -3 ${O}_full.log
ls -la gpurun_out/ | grep r2ca
