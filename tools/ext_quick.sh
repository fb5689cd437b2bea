cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/sps_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sps_tests.log
export RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 MASTER_ADDR=127.0.0.1 MASTER_PORT=29655
for i in 1 2; do
timeout -s KILL 300 python bench.py --sp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sp1_plain.log 2>&1
python -c "
import json
for l in open('gpurun_out/sp1_plain.log'):
    if l.startswith('{'): d=json.loads(l); print('sp1', d['value'], d['ms_per_step'], d['a2a'])
"
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pl.log 2>&1
python -c "
import json
for l in open('gpurun_out/pl.log'):
    if l.startswith('{'): d=json.loads(l); print('plain', d['value'], d['ms_per_step'])
"
done
