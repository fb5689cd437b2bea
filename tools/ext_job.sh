cd $GRAFT_REPO_ROOT
timeout -s KILL 400 python -m pytest tests/test_gpu_ext.py -x -q > gpurun_out/ext_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ext_tests.log
timeout -s KILL 300 python tools/ext_bench.py > gpurun_out/ext_bench.log 2>&1; echo "rc=$?" >> gpurun_out/ext_bench.log
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/ext_all_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ext_all_gpu.log
timeout -s KILL 300 python bench.py --no-cpu-baseline > gpurun_out/ext_headline.log 2>&1; echo "rc=$?" >> gpurun_out/ext_headline.log
