#!/bin/bash
# A/B of two library builds on the bench workload, alternated in one box session.
#   A=paper_2510_21270_b200/libpbs_b200.so B=build/ab_old/libpbs_b200.so bash scripts/ab_attn.sh [bench args]
A=${A:-paper_2510_21270_b200/libpbs_b200.so}
B=${B:-build/ab_old/libpbs_b200.so}
mkdir -p gpurun_out/ab
for r in 1 2 3; do
  for lib in "$A" "$B"; do
    PBS_B200_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab/run.json 2>/dev/null
    python scripts/ab_line.py "$lib" gpurun_out/ab/run.json
  done
done
