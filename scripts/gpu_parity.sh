#!/bin/bash
# On the GPU box: the bench-config parity against the compiled reference, the
# exhaustive expf test, then the whole GPU suite; audits into gpurun_out/audit.
export PBS_AUDIT_DIR=gpurun_out/audit
mkdir -p gpurun_out/audit
nproc > gpurun_out/audit/nproc.txt
lscpu > gpurun_out/audit/lscpu.txt 2>&1
python -m pytest tests/test_fullsize_parity.py tests/test_expf.py -x -q -s -m gpu 2>&1 | tail -30 > gpurun_out/audit/new_tests.log
python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/audit/gpu_suite.log
cat gpurun_out/audit/new_tests.log gpurun_out/audit/gpu_suite.log
