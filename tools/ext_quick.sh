cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python tools/gap_probe.py > gpurun_out/gap.log 2>&1; echo "rc=$?" >> gpurun_out/gap.log
