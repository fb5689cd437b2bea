cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_gpu_ext.py -x -q > gpurun_out/x_tests.log 2>&1; echo "rc=$?" >> gpurun_out/x_tests.log
timeout -s KILL 300 python tools/ext_bench.py > gpurun_out/x_bench.log 2>&1
