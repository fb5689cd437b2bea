cd $GRAFT_REPO_ROOT
for c in 1 3 4 5; do S=10; [ $c = 3 ] && S=3; timeout -s KILL 600 python bench.py --config $c --steps $S --warmup 3 > gpurun_out/r1h_cfg$c.log 2>&1; echo "rc=$?" >> gpurun_out/r1h_cfg$c.log; done
