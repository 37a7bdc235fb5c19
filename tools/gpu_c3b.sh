cd $GRAFT_REPO_ROOT
for inf in 0 6400 12800; do
timeout 900 python tools/bench_configs.py c3 --rounds 8 --seq-rounds 0 --inflight $inf > gpurun_out/c3b_i$inf.log 2>&1; echo "inflight $inf rc=$?"
done
