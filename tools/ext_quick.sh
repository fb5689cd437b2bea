cd $GRAFT_REPO_ROOT
for i in 1 2; do
for bn in 256 240 208; do
VC_QKV_BN=$bn timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/c_b.log 2>&1
python - $bn <<'PY'
import json,sys
for l in open("gpurun_out/c_b.log"):
    if l.startswith("{"):
        d=json.loads(l); s=d["block"]["stage_ms"]
        print("bn", sys.argv[1], "ms %.3f"%d["ms_per_step"], "qkv %.4f"%s["qkv_gemm"])
PY
done; done
