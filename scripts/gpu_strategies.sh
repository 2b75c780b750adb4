cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for s in query_permute both; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --strategy $s 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$s', d['value'], d['e2e']['value'], d['stage_ms'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"query_group|centroid|qnorm|segmented|block_logits|importance" -c 40 --csv --log-file gpurun_out/launches_qp.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --strategy query_permute > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/launches_qp.csv 2>&1 | head -12
