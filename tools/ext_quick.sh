cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout -s KILL 120 tools/_bin/attn_trace 21600 1350 24 66 0 10 | head -1 | sed "s/^/base /"
timeout -s KILL 120 tools/_bin/attn_trace_cs 21600 1350 24 66 0 10 | head -1 | sed "s/^/cs /"
timeout -s KILL 120 tools/_bin/attn_trace 21600 21856 24 66 256 3 | head -1 | sed "s/^/base /"
timeout -s KILL 120 tools/_bin/attn_trace_cs 21600 21856 24 66 256 3 | head -1 | sed "s/^/cs /"
done
