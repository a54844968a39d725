#!/bin/bash
# A/B: CE ring pass 2, A = per-vector bounds checks in pass 2, B = whole pieces specialised
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
cp $L/ab/libB.so $L/libliger_b200.so
timeout 900 python -m pytest tests/test_gpu_ce.py tests/test_gpu_flce.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/r2av_ab.log
for r in 1 2; do for v in A B; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v: $(python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), {k: round(v, 3) for k, v in d["roofline"]["stage_ms_per_step"].items()}, d["clocks"]["sm_mhz"])')" >> gpurun_out/r2av_ab.log
  echo "$v ce: $(python bench_kernels.py --only cross_entropy 2>&1 | tail -1)" >> gpurun_out/r2av_ab.log
done; done
cat gpurun_out/r2av_ab.log
