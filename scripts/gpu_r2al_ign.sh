#!/bin/bash
# finalize stage time vs ignored-target fraction (row imbalance of the static round-robin ring)
cd "$GRAFT_REPO_ROOT"
for r in 1 2; do for f in 0.0 0.1 0.3; do
  echo "ignore $f: $(python bench.py --steps 20 --warmup 5 --ignore-frac $f --no-cpu-baseline --no-variants 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), {k: round(v, 3) for k, v in d["roofline"]["stage_ms_per_step"].items()}, d["clocks"]["sm_mhz"])')" >> gpurun_out/r2al.log
done; done
timeout 900 python -m pytest tests/test_gpu_distributed.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2al.log
cat gpurun_out/r2al.log
