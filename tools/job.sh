#!/bin/bash
# One parameterised GPU job (replaces the per-run r1*_job.sh scripts):
#   gpurun -- 'bash tools/job.sh TAG step [step ...]'
# steps: tests smoke bench ref sp1 launches ncufull ext cfgN (bench --config N)
# Logs go to gpurun_out/TAG_<step>.log with the exit code appended.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=$1; shift
run() {  # run LIMIT NAME CMD...
  local lim=$1 name=$2; shift 2
  timeout -s KILL "$lim" "$@" > "gpurun_out/${TAG}_${name}.log" 2>&1
  echo "rc=$?" >> "gpurun_out/${TAG}_${name}.log"
}
for step in "$@"; do
  case $step in
    tests) run 1200 tests python -m pytest tests -m gpu -x -q ;;
    smoke) run 300 smoke python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" ;;
    bench) run 400 bench python bench.py ;;
    ref) run 400 ref python bench.py --impl reference ;;
    sp1) run 300 sp1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
           --master-port 29631 bench.py --gpus 1 --steps 5 --warmup 3 --sp ;;
    launches) run 300 launches ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
           --log-file "gpurun_out/${TAG}_launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline ;;
    ncufull) run 900 ncufull ncu --set full --clock-control none --import-source on \
           -k regex:"ln_rows|gemm_tc|attn_t|temporal" -c 10 -o "gpurun_out/${TAG}_block" python tools/run_block.py --iters 1 ;;
    ext) run 300 ext python tools/ext_bench.py ;;
    cfg*) run 600 "$step" python bench.py --config "${step#cfg}" --no-cpu-baseline ;;
    py:*) run 900 "$(echo "${step#py:}" | tr -c 'a-zA-Z0-9_\n' '_' | cut -c1-40)" python ${step#py:} ;;
    *) echo "unknown step $step" ;;
  esac
done
