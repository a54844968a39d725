#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python scripts/determinism_stage.py > gpurun_out/r2f_det.log 2>&1
cat gpurun_out/r2f_det.log | cut -c1-600
