#!/bin/bash
# Round profile refresh: GPU tests, smoke, C3 bench, Qwen C4 bench, density sweep,
# launch list, one full attention capture, captures of the other stages.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
bash scripts/gpu_check.sh > gpurun_out/check.log 2>&1
timeout 900 python bench.py --model qwen > gpurun_out/bench_qwen.log 2>&1; echo "qwen rc=$?" >> gpurun_out/bench_qwen.log
timeout 900 python scripts/density_sweep_bench.py > gpurun_out/density_sweep.jsonl 2> gpurun_out/density_sweep.err
bash scripts/gpu_ncu_multi.sh
ls -la gpurun_out
