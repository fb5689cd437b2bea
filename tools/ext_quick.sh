cd $GRAFT_REPO_ROOT
VC_ATTN_PERSIST=2 timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p_tests.log
tail -3 gpurun_out/p_tests.log
VC_ATTN_PERSIST=2 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/p_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/p_tests2.log
tail -3 gpurun_out/p_tests2.log
for i in 1 2 3; do
for pm in 0 1; do
VC_ATTN_PERSIST=$pm timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/p_b.log 2>&1
python - $pm <<'PY'
import json,sys
for l in open("gpurun_out/p_b.log"):
    if l.startswith("{"):
        d=json.loads(l); s=d["block"]["stage_ms"]
        print("persist", sys.argv[1], "ms %.3f"%d["ms_per_step"], "spatial %.4f fs %.4f"%(s["attn_spatial"], s["attn_fullseq"]))
PY
done; done
