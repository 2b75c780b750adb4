#!/bin/bash
# Round profile refresh: GPU tests, smoke, C3 bench, launch list, one full attention
# capture (gpu_check.sh), Qwen C4 and C2 32K bench lines, the B = 64 variant, the
# density sweep, the strategies at 128K, and captures of the other stages.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
bash scripts/gpu_check.sh > gpurun_out/check.log 2>&1
timeout 900 python bench.py --model qwen > gpurun_out/bench_qwen.log 2>&1; echo "qwen rc=$?" >> gpurun_out/bench_qwen.log
timeout 900 python bench.py --seq 32768 > gpurun_out/bench_c2.log 2>&1; echo "c2 rc=$?" >> gpurun_out/bench_c2.log
timeout 900 python bench.py --block 64 --no-cpu-baseline > gpurun_out/bench_b64.log 2>&1; echo "b64 rc=$?" >> gpurun_out/bench_b64.log
timeout 900 python scripts/density_sweep_bench.py > gpurun_out/density_sweep.jsonl 2> gpurun_out/density_sweep.err
for s in both query_permute none; do
  timeout 900 python bench.py --strategy $s --no-cpu-baseline --no-e2e > gpurun_out/bench_$s.log 2>&1
done
bash scripts/gpu_ncu_multi.sh
ls -la gpurun_out
