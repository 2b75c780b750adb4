cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 120 -k "host_entry" 2>&1 | tail -3
