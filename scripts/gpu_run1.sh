python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['dense_fa_ms'], d['stage_ms'], d['roofline']['frac'], d['clocks'])"; done
python bench.py --model qwen --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('qwen', d['value'], d['e2e']['value'], d['stage_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select" -c 20 --csv --log-file gpurun_out/launches_sel.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/launches_sel.csv 2>&1 | head -4
