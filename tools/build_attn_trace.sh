#!/bin/bash
# Build tools/_bin/attn_trace: every csrc/*.cu with -DVC_ATTN_TRACE plus the
# driver in tools/attn_trace.cu (a profiling aid, not part of the library).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/tools/_bin
mkdir -p "$OUT"
EXTRA=${EXTRA:-}
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  --expt-relaxed-constexpr -DVC_ATTN_TRACE -DVC_TUNING $EXTRA -I "$ROOT/include" \
  "$ROOT"/paper_2501_08453_b200/csrc/*.cu "$ROOT/tools/attn_trace.cu" -o "$OUT/attn_trace${SUFFIX:-}" -lcuda
echo "built $OUT/attn_trace${SUFFIX:-}"
