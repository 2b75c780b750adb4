timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_properties.py -q -x -m gpu 2>&1 | tail -3
cd scripts; PBS_B200_LIB=../build/events/libpbs_b200.so timeout 300 python attn_events.py 2>&1 | tail -10; cd ..
for r in 1 2; do
for v in prod maxfirst base; do
  lib=build/$v/libpbs_b200.so; [ $v = prod ] && lib=paper_2510_21270_b200/libpbs_b200.so
  PBS_B200_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_run.json 2>/dev/null
  python scripts/ab_line.py "$v/x" gpurun_out/ab_run.json
done
done
