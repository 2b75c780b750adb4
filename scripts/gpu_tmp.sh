cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 120 -k "tiny_and_ragged or selection_extremes" 2>&1 | tail -4
