#!/bin/bash
# compute-sanitizer on the box: smoke under memcheck / synccheck / racecheck, then
# memcheck over the GPU parity, tensor-I/O and workload suites.  Output: gpurun_out/sanitizer.txt
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
out=gpurun_out/sanitizer.txt
echo "# compute-sanitizer on the B200 box (round 2, final tree)" > $out
echo "## smoke() under memcheck / synccheck / racecheck" >> $out
for tool in memcheck synccheck racecheck; do
  echo "== $tool" >> $out
  timeout 900 compute-sanitizer --tool $tool python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | grep -E "COMPUTE-SANITIZER|smoke|SUMMARY|Error|error" | head -20 >> $out
done
echo "## memcheck over tests/test_gpu_parity.py + test_tensor_io.py + test_workload.py (-m gpu, fullsize tests excluded)" >> $out
timeout 2400 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_tensor_io.py tests/test_workload.py -q -m gpu -p no:cacheprovider 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|SUMMARY|Invalid|error" | head -30 >> $out
cat $out
