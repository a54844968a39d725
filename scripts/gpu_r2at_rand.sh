#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_flce.py -m gpu -q -p no:cacheprovider -k "random_configs" 2>&1 | tail -15
