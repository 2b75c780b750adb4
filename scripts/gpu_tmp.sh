cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/abnew
for r in 1 2; do
for lib in build/r88/libpbs_b200.so build/ispin/libpbs_b200.so build/sspin/libpbs_b200.so build/ispin_sspin/libpbs_b200.so; do
  PBS_B200_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/abnew/run.json 2>/dev/null
  python scripts/ab_line.py "$lib" gpurun_out/abnew/run.json
done; done
