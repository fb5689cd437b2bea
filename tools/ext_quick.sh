cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python bench.py --no-cpu-baseline > gpurun_out/clk.log 2>&1
python -c "
import json
for l in open('gpurun_out/clk.log'):
    if l.startswith('{'): d=json.loads(l); print(d['clocks'], d['ms_per_step'], d['steps'])
"
python - <<'PY'
import time, pynvml
pynvml.nvmlInit(); h=pynvml.nvmlDeviceGetHandleByIndex(0)
t=time.time(); n=0
while time.time()-t<0.2:
    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM); pynvml.nvmlDeviceGetCurrentClocksEventReasons(h); n+=1
print("nvml sample pairs per second:", n/0.2)
PY
