cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest tests/test_workload.py tests/test_tensor_io.py -x -q -m gpu --timeout 300 2>&1 | tail -4
