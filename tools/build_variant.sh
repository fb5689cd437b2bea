#!/bin/bash
# Build a variant of the library with extra nvcc flags into tools/_bin/NAME/
# (for interleaved A/B on one box: VC_LIB_PATH=tools/_bin/NAME/libvchitect_b200.so).
#   bash tools/build_variant.sh NAME -DFLAG ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/tools/_bin/$NAME
mkdir -p "$OUT"
for f in "$ROOT"/paper_2501_08453_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I "$ROOT/include" "$@" -c "$f" -o "$OUT/$(basename "$f" .cu).o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libvchitect_b200.so" "$OUT"/*.o
echo "built $OUT/libvchitect_b200.so"
