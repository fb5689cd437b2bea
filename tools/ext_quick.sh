cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/ln_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ln_tests.log
for i in 1 2; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ln_b.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/ln_b.log"):
    if l.startswith("{"):
        d=json.loads(l); s=d["block"]["stage_ms"]
        print("ms %.3f"%d["ms_per_step"], " ".join("%s %.3f"%(k,v) for k,v in s.items()))
PY
done
