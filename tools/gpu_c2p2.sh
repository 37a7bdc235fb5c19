cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for lanes in 0 16 2064 2080 1288; do
timeout 600 python tools/bench_configs.py c2p --rounds 8 --seq-rounds 1 --no-cpu --lanes $lanes > gpurun_out/c2p2_l${lanes}_$rep.log 2>&1; echo "c2p lanes $lanes rc=$?"
done; done
for lanes in 0 16 2064 2080; do
timeout 600 python tools/bench_configs.py c4 --rounds 6 --cache-flags 3 --lanes $lanes > gpurun_out/c4l_l$lanes.log 2>&1; echo "c4 lanes $lanes rc=$?"
done
