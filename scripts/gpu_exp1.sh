# softmax-chain experiments: spans of the product, of a no-op softmax and of a load+max-only softmax
for v in spans spansnop spansload; do
  PBS_B200_LIB=build/$v/libpbs_b200.so timeout 300 python scripts/attn_trace.py --spans > gpurun_out/spans_$v.txt 2>&1
done
paste gpurun_out/spans_spans.txt gpurun_out/spans_spansnop.txt gpurun_out/spans_spansload.txt
for lib in paper_2510_21270_b200/libpbs_b200.so build/nop/libpbs_b200.so; do
  PBS_B200_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_run.json 2>/dev/null
  python scripts/ab_line.py "$lib" gpurun_out/ab_run.json
done
