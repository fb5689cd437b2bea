cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_bench_contract.py -x -q > gpurun_out/bc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bc_tests.log
