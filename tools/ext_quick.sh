cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=temperature.gpu,power.draw,clocks.sm,power.limit --format=csv
for i in 1 2 3 4; do
for lib in tools/_bin/lib_88dfe05.so paper_2501_08453_b200/libvchitect_b200.so; do
VC_LIB_PATH=$PWD/$lib timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab.log 2>&1
python - "$lib" <<'PY'
import json,sys
for l in open("gpurun_out/ab.log"):
    if l.startswith("{"):
        d=json.loads(l); s=d["block"]["stage_ms"]
        print(sys.argv[1][-20:], "ms %.3f"%d["ms_per_step"], "sum %.3f"%sum(s.values()), "qkv %.3f sp %.3f fs %.3f"%(s["qkv_gemm"],s["attn_spatial"],s["attn_fullseq"]), "clk", d["clocks"]["sm_mhz"], "e2e %.0f"%d["e2e"]["value"])
PY
done; done
nvidia-smi --query-gpu=temperature.gpu,power.draw,clocks.sm,power.limit --format=csv
