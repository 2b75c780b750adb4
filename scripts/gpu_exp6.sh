timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -2
for r in 1 2; do
for v in prod base s32 s200 nopp poly2; do
  lib=build/$v/libpbs_b200.so; [ $v = prod ] && lib=paper_2510_21270_b200/libpbs_b200.so
  PBS_B200_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_run.json 2>/dev/null
  python scripts/ab_line.py "$v/x" gpurun_out/ab_run.json
done
done
