#!/bin/bash
# Staged target-range check (host waits for the count kernel only): full GPU suite, then the
# bench (value vs e2e) twice.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2ax
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_gputests.log 2>&1
tail -3 ${O}_gputests.log
for r in 1 2; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | tail -1 >> ${O}_bench.jsonl
done
python -c "
import json
for l in open('${O}_bench.jsonl'):
    d=json.loads(l); print(round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'])"
