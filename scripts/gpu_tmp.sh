cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/abnew
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -x -q -m gpu --timeout 600 -k "importance or pipeline_matches or c2 or host_entry or fixtures" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:importance -c 12 --csv --log-file gpurun_out/abnew/l.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/abnew/l.csv 2>&1 | head -8
for r in 1 2; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/abnew/run.json 2>/dev/null; python scripts/ab_line.py "x/fused/y" gpurun_out/abnew/run.json
  PBS_EXP_SEPARATE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/abnew/run.json 2>/dev/null; python scripts/ab_line.py "x/separate/y" gpurun_out/abnew/run.json
done
