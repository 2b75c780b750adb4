#!/bin/bash
# On the GPU box: the GPU suite file by file, each test bounded by pytest-timeout,
# verbose logs under gpurun_out/suite/ (readable even if the call is cut off).
#   bash scripts/gpu_suite.sh [test files...]
export PBS_AUDIT_DIR=gpurun_out/audit
mkdir -p gpurun_out/suite gpurun_out/audit
FILES=${@:-$(ls tests/test_*.py)}
for f in $FILES; do
  name=$(basename $f .py)
  timeout 1200 python -m pytest $f -q -m gpu --timeout 600 -rf --durations=15 > gpurun_out/suite/$name.log 2>&1
  echo "$name rc=$? $(tail -1 gpurun_out/suite/$name.log)"
done
