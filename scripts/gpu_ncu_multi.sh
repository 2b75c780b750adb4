#!/bin/bash
# ncu --set full captures of the non-attention stages (one launch each) from a short bench run
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for k in ${NCU_KERNELS:-importance_logits importance_exp importance_denom importance_scores select_warp apply_rows pool_bf16}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/prof_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$k.log 2>&1
done
