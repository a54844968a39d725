#!/bin/bash
# After the device-count GEMM limits: full GPU suite, smoke, memcheck of the device-count
# kept-row path, and the default bench.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2bw
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_gputests.log 2>&1
tail -1 ${O}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 10 python -m pytest tests/test_gpu_compact.py -q -p no:cacheprovider -k "device_count and (default or _frac or reduction)" > ${O}_memcheck.log 2>&1; echo "memcheck rc=$?"
grep -E "ERROR SUMMARY|passed|failed" ${O}_memcheck.log | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > ${O}_bench.jsonl
python -c "
import json; d=json.loads(open('${O}_bench.jsonl').read()); r=d['roofline']
print(round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], round(r['frac'],3))"
