#!/bin/bash
# round-2 GPU check: full -m gpu suite (durations) + smoke
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/r2_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
tail -3 gpurun_out/r2_gputests.log; tail -2 gpurun_out/r2_smoke.log
