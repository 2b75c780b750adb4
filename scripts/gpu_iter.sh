#!/bin/bash
# On the GPU box: the GPU parity suite, then a short bench line (no CPU baseline).
#   scripts/gpu_iter.sh [pytest selection] [bench args]
SEL=${1:-tests/test_gpu_parity.py}
shift
mkdir -p gpurun_out/iter
timeout 900 python -m pytest $SEL -x -q -m gpu 2>&1 | tail -25 > gpurun_out/iter/tests.log
cat gpurun_out/iter/tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/iter/bench.json 2> gpurun_out/iter/bench.err
tail -3 gpurun_out/iter/bench.err
python -c "
import json; d=json.load(open('gpurun_out/iter/bench.json'))
print('value', d['value'], 'e2e', d['e2e'] and d['e2e']['value'], 'dense', d['dense_fa_ms'], 'stage', d['stage_ms'], 'frac', d['roofline']['frac'], 'clk', d['clocks'])"
