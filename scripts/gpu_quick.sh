#!/bin/bash
# Quick box check: GPU tests and three C3 bench lines (value, e2e, dense FA, attention stage, roofline, clocks).
cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['dense_fa_ms'], d['stage_ms']['attention'], d['roofline']['frac'], d['clocks'])"; done
