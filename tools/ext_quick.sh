cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/all_tests.log 2>&1; echo "rc=$?" >> gpurun_out/all_tests.log
