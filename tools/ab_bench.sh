#!/bin/bash
# Same-box A/B of tuning switches through the real block bench:
#   gpurun -- 'bash tools/ab_bench.sh TAG ROUNDS "VAR=a" "VAR=b" ...'
# Builds the library with -DVC_TUNING (vc_tuning.h reads VC_* from the
# environment), then runs bench.py config 2 once per variant per round,
# interleaved, and prints ms_per_step and the per-stage times.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=$1; ROUNDS=$2; shift 2
[ -n "$AB_NOBUILD" ] || python -m paper_2501_08453_b200.build --force --tuning > "gpurun_out/${TAG}_build.log" 2>&1 || { echo build failed; exit 1; }
for r in $(seq "$ROUNDS"); do
  for v in "$@"; do
    env $v timeout 300 python bench.py --no-cpu-baseline --steps 20 ${AB_ARGS:-} 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); s = d['block']['stage_ms']
        print('$v', round(d['ms_per_step'], 4), ' '.join(f'{k}={v:.4f}' for k, v in s.items()))
"
  done
done | tee "gpurun_out/${TAG}_ab.log"
