cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/abnew
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 120 -k "host_entry or c1_config or dist or shard" > gpurun_out/abnew/tests.log 2>&1
tail -3 gpurun_out/abnew/tests.log
timeout 300 python scripts/e2e_probe.py > gpurun_out/abnew/e2e.txt 2>&1
cat gpurun_out/abnew/e2e.txt | tail -36 | head -12
for i in 1 2 3; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dense 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['stage_ms']['attention'], d['clocks']['sm_mhz'])"; done
