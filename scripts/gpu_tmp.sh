cd "${GRAFT_REPO_ROOT:-.}"
python scripts/pcie_probe.py 2>&1 | tail -2
python scripts/e2e_trace.py 32768 2>&1 | tail -40
