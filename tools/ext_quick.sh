cd $GRAFT_REPO_ROOT
for i in 1 2; do
for lib in lib_t0 lib_t5 lib_t6; do
VC_LIB_PATH=$PWD/tools/_bin/$lib.so timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/t_b.log 2>&1
python - $lib <<'PY'
import json,sys
for l in open("gpurun_out/t_b.log"):
    if l.startswith("{"):
        d=json.loads(l); s=d["block"]["stage_ms"]
        print(sys.argv[1], "ms %.3f"%d["ms_per_step"], "temporal %.4f"%s["attn_temporal"])
PY
done; done
