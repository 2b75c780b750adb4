cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/abnew
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 -k "query or both or pipeline_matches or host_entry or tiny" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"query_group|centroid|qnorm" -c 14 --csv --log-file gpurun_out/abnew/l.csv python bench.py --strategy both --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/abnew/l.csv 2>&1 | head -7
for lib in build/r88/libpbs_b200.so paper_2510_21270_b200/libpbs_b200.so; do
  PBS_B200_LIB=$lib timeout 300 python bench.py --strategy both --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/abnew/run.json 2>/dev/null
  python scripts/ab_line.py "$lib" gpurun_out/abnew/run.json
done
