cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r2final
bash tools/job.sh $T smoke bench ref
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_ncu_launch.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"ln_rows|gemm_tc|attn_t|temporal|fill_vt" -c 10 -o gpurun_out/${T}_block python tools/run_block.py --iters 1 > gpurun_out/${T}_ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_ncu_full.log
bash tools/job.sh $T cfg1 cfg5 cfg3 cfg4
