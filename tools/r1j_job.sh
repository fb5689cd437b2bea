cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1j_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r1j_gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1j_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r1j_smoke.log
timeout -s KILL 400 python bench.py > gpurun_out/r1j_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r1j_bench.log
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/r1j_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r1j_bench_ref.log
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 1 --steps 5 --warmup 3 --sp > gpurun_out/r1j_sp1.log 2>&1; echo "rc=$?" >> gpurun_out/r1j_sp1.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1j_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1j_ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/r1j_ncu_launch.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"ln_rows|gemm_tc|attn_tc|temporal" -c 7 -o gpurun_out/r1j_block python tools/run_block.py --iters 1 > gpurun_out/r1j_ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/r1j_ncu_full.log
timeout -s KILL 300 python tools/ext_bench.py > gpurun_out/r1j_ext_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r1j_ext_bench.log
