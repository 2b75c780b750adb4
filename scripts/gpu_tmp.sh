cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/abnew
PBS_B200_LIB=build/chunk64/libpbs_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 120 -k "pipeline_matches_oracle or many_items or dense or tiny or coverage" 2>&1 | tail -3
for r in 1 2; do
for lib in build/r88/libpbs_b200.so build/chunk64/libpbs_b200.so build/chunk64p4/libpbs_b200.so; do
  PBS_B200_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abnew/run.json 2>/dev/null
  python scripts/ab_line.py "$lib" gpurun_out/abnew/run.json
done; done
