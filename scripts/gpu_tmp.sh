cd "${GRAFT_REPO_ROOT:-.}"
export PBS_AUDIT_DIR=gpurun_out/audit
timeout 900 python -m pytest tests/test_fullsize_parity.py -x -q -m gpu --timeout 600 -k "b64 or c2" -s 2>&1 | grep -E "^\{|passed|failed|Error" | head
