#!/bin/bash
# Runs HERE (needs /root/reference): the reference's own CPU bench for a few ops, merged with the
# GPU records of `python -m paper_2410_10989_b200.benchrecord --dtype f32 ...` (profiles/), and
# summarised by the reference's own `rowfuse report` (rowfuse/cli.py:275-289).
set -e
cd /root/repo
PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python -m rowfuse.cli bench \
  --ops rmsnorm,layernorm,swiglu,geglu,rope,cross_entropy,linear_ce --repeats 3 --dtype f32 --csv /tmp/ref_bench.csv > /dev/null
python - <<'PY'
import csv
ref = list(csv.reader(open("/tmp/ref_bench.csv")))
gpu = list(csv.reader(open("profiles/r02/r2_benchrecord_gpu_f32.csv")))
rows = [r for r in ref[1:] if r[1] == "reference"] + gpu[1:]
with open("/tmp/merged_bench.csv", "w", newline="") as f:
    w = csv.writer(f); w.writerow(ref[0]); w.writerows(rows)
PY
PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python -m rowfuse.cli report /tmp/merged_bench.csv
