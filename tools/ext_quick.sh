cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_gpu_sp.py -x -q > gpurun_out/sp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sp_tests.log
export RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 MASTER_ADDR=127.0.0.1 MASTER_PORT=29655
timeout -s KILL 300 python bench.py --sp --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sp1_plain.log 2>&1; echo "rc=$?" >> gpurun_out/sp1_plain.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sp1_launches.csv python bench.py --sp --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/sp1_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/sp1_ncu.log
