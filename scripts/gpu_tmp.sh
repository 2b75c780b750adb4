cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/abnew
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -x -q -m gpu --timeout 300 -k "pipeline_matches or many_items or tiny or extremes or shards or host_entry or b64" 2>&1 | tail -1
for lib in build/r88/libpbs_b200.so paper_2510_21270_b200/libpbs_b200.so; do
  PBS_B200_LIB=$lib timeout 300 python bench.py --block 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/abnew/run.json 2>/dev/null
  python scripts/ab_line.py "$lib" gpurun_out/abnew/run.json
  PBS_B200_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/abnew/run.json 2>/dev/null
  python scripts/ab_line.py "$lib" gpurun_out/abnew/run.json
done
