cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:importance_logits -c 6 --csv --log-file gpurun_out/launches_lg.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/launches_lg.csv 2>&1 | head -3
