# A/B of attention variants on the bench workload (two passes, alternated)
for r in 1 2; do
for v in prod late v3 k3 poly2 poly4 nop nopnokv nopv3; do
  lib=build/$v/libpbs_b200.so; [ $v = prod ] && lib=paper_2510_21270_b200/libpbs_b200.so
  PBS_B200_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/ab_run.json 2>/dev/null
  python scripts/ab_line.py "$v/x" gpurun_out/ab_run.json
done
done
