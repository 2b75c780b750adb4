#!/bin/bash
# Build a variant of libpbs_b200.so with extra nvcc flags into build/<name>/ (A/B and debug builds):
#   bash scripts/build_variant.sh spans -DPBS_ATTN_SPANS
#   PBS_B200_LIB=build/spans/libpbs_b200.so python ...
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/$NAME
mkdir -p "$OUT"
for f in "$ROOT"/paper_2510_21270_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I "$ROOT/include" -I "$ROOT/paper_2510_21270_b200/csrc" "$@" \
    -c "$f" -o "$OUT/$(basename "${f%.cu}").o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libpbs_b200.so" "$OUT"/*.o -lcudart_static
echo "$OUT/libpbs_b200.so"
