cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | grep -E "SUMMARY|Error|smoke" | head
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 120 -k "pipeline_matches_oracle or many_items" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms']['attention'], d['clocks']['sm_mhz'])"; done
