cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/final3
export PBS_AUDIT_DIR=gpurun_out/final3/audit
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/final3/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final3/gpu_tests.log
tail -3 gpurun_out/final3/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
