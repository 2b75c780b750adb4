cd "${GRAFT_REPO_ROOT:-.}"
PBS_LOGITS_W2=1 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "importance or pipeline or host_entry" 2>&1 | tail -2
for w in "" 1; do
PBS_LOGITS_W2=$w timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:importance_logits -c 6 --csv --log-file gpurun_out/launches_lg$w.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/launches_lg$w.csv 2>&1 | sed -n 2p
done
