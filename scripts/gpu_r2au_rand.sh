#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_random.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -25
