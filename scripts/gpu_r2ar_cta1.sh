#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_flce.py -m gpu -q -p no:cacheprovider -k "single_cta or different_devices" 2>&1 | tail -3
