cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/abnew
PBS_B200_LIB=build/gpre1/libpbs_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 120 -k "importance" 2>&1 | tail -1
for lib in build/r88/libpbs_b200.so build/gpre1/libpbs_b200.so build/g1/libpbs_b200.so; do
  PBS_B200_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:importance_logits -c 6 --csv --log-file gpurun_out/abnew/l.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
  echo $lib; python profiles/summarize_launches.py gpurun_out/abnew/l.csv 2>&1 | sed -n 2p
done
