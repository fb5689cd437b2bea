cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_attention.py tests/test_gpu_parity.py > gpurun_out/r2au_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2au_tests.log
for i in 1 2; do for b in attn_trace attn_trace_np; do echo $b >> gpurun_out/r2au.log; timeout -s KILL 60 tools/_bin/$b 21600 21856 24 66 256 10 | head -1 >> gpurun_out/r2au.log; timeout -s KILL 60 tools/_bin/$b 1350 1350 384 66 0 10 | head -1 >> gpurun_out/r2au.log; done; done
