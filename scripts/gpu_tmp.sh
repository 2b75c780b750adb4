cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/abnew
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 -k "query or both or pipeline_matches or host_entry or tiny" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum --clock-control none -k regex:"query_group_screen" -c 2 --csv --log-file gpurun_out/abnew/l.csv python bench.py --strategy both --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/abnew/l.csv')) if len(r)>10]
h=rows[0]; iN=h.index('Kernel Name'); iM=h.index('Metric Name'); iV=h.index('Metric Value')
for r in rows[1:]: print(r[iN][:45], r[iM], r[iV])
"
for lib in build/r88/libpbs_b200.so paper_2510_21270_b200/libpbs_b200.so; do
  PBS_B200_LIB=$lib timeout 300 python bench.py --strategy both --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/abnew/run.json 2>/dev/null
  python scripts/ab_line.py "$lib" gpurun_out/abnew/run.json
done
