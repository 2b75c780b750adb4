cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/final2
export PBS_AUDIT_DIR=gpurun_out/final2/audit
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/final2/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final2/gpu_tests.log
tail -3 gpurun_out/final2/gpu_tests.log
for s in both query_permute; do
  timeout 900 python bench.py --strategy $s --no-cpu-baseline --no-e2e > gpurun_out/final2/bench_$s.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final2/launches_both.csv python bench.py --strategy both --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/final2/launches_both.csv > gpurun_out/final2/launches_both.txt 2>&1; head -12 gpurun_out/final2/launches_both.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_group_screen -c 1 -o gpurun_out/final2/prof_qscreen -f python bench.py --strategy both --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
python profiles/summarize_ncu.py gpurun_out/final2/prof_qscreen.ncu-rep > gpurun_out/final2/ncu_qscreen.txt 2>&1
