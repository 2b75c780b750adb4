cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 -k "query or both or pipeline_matches or host_entry or tiny" 2>&1 | tail -1
timeout 900 compute-sanitizer --tool racecheck python -c "
import torch
from paper_2510_21270_b200 import ops
g=torch.Generator().manual_seed(0)
q=torch.randn(4,2048+77,128,generator=g).bfloat16().cuda(); k=torch.randn(2,2048+77,128,generator=g).bfloat16().cuda(); v=torch.randn(2,2048+77,128,generator=g).bfloat16().cuda()
r=ops.pbs_attention(q,k,v,ops.make_config(strategy='both')); print('both ok', r.report['selected_blocks'])
" 2>&1 | grep -E "ok|SUMMARY|Error" | head -4
for i in 1 2; do timeout 300 python bench.py --strategy both --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-dense 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms']['estimate'])"; done
