python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/e2e_probe.py 2>&1 | tail -5
for i in 1 2; do python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['stage_ms']['attention'], d['clocks'])"; done
python bench.py --model qwen --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('qwen', d['value'], d['e2e']['value'], d['stage_ms'])"
