cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/b64
timeout 600 python bench.py --block 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b64/b64.json 2>gpurun_out/b64/b64.err; tail -2 gpurun_out/b64/b64.err
python -c "import json; d=json.load(open('gpurun_out/b64/b64.json')); print('b64', d['value'], d['stage_ms'], d['block_density'], d['roofline']['achieved'], d['dense_fa_ms'])"
timeout 600 python bench.py --block 64 --seq 32768 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b64/b64_32k.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b64/b64_32k.json')); print('b64 32k', d['value'], d['stage_ms'], d['block_density'])"
PBS_FORCE_SIMT=1 timeout 900 python bench.py --block 64 --seq 32768 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b64/b64_32k_simt.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b64/b64_32k_simt.json')); print('b64 32k simt', d['value'], d['stage_ms'])"
timeout 600 python bench.py --seq 32768 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b64/b128_32k.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b64/b128_32k.json')); print('b128 32k', d['value'], d['stage_ms'], d['block_density'])"
