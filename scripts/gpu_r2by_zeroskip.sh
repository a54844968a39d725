#!/bin/bash
# Unread ignored-slot zero writes skipped in the finalize (device count): full GPU suite, the
# kept-count probe, memcheck of the device-count special paths.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2by
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_gputests.log 2>&1
tail -1 ${O}_gputests.log; grep FAILED ${O}_gputests.log | head -5
timeout -s KILL 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 10 python -m pytest tests/test_gpu_compact.py -q -p no:cacheprovider -k "special_paths" > ${O}_memcheck.log 2>&1; echo "memcheck rc=$?"
grep -E "ERROR SUMMARY|passed|failed" ${O}_memcheck.log | tail -2
timeout 600 python scripts/kept_count_probe.py 10 2>&1 | tail -3
