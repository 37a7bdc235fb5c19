cd $GRAFT_REPO_ROOT
for lanes in 0 2080 16 2056 1288; do
timeout 600 python tools/bench_configs.py c2p --rounds 8 --seq-rounds 1 --no-cpu --lanes $lanes > gpurun_out/c2p_l$lanes.log 2>&1; echo "lanes $lanes rc=$?"
done
