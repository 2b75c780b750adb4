#!/bin/bash
# One full ncu capture of one kernel launch from a short bench run (no timing use).
#   NCU_KERNEL=attn_sm100 NCU_SKIP=0 BENCH_ARGS="--seq 131072" bash scripts/gpu_ncu.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout ${NCU_TIMEOUT:-1200} ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-attn_sm100} \
  -s ${NCU_SKIP:-0} -c 1 -o gpurun_out/${NCU_OUT:-prof} -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
