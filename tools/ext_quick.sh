cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s_tests.log
for i in 1 2 3; do
for lib in tools/_bin/lib_prev.so paper_2501_08453_b200/libvchitect_b200.so; do
VC_LIB_PATH=$PWD/$lib timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/s_b.log 2>&1
python - $lib <<'PY'
import json,sys
for l in open("gpurun_out/s_b.log"):
    if l.startswith("{"):
        d=json.loads(l); s=d["block"]["stage_ms"]
        print(sys.argv[1][-22:], "ms %.3f"%d["ms_per_step"], "tm %.4f"%s["attn_temporal"], "sum %.3f"%sum(s.values()))
PY
done; done
