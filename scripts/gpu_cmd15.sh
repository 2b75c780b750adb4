PBS_B200_LIB=build/spans/libpbs_b200.so python scripts/attn_trace.py --spans > gpurun_out/spans_base.txt 2>&1
PBS_B200_LIB=build/spansfake/libpbs_b200.so python scripts/attn_trace.py --spans > gpurun_out/spans_fake.txt 2>&1
paste gpurun_out/spans_base.txt gpurun_out/spans_fake.txt
