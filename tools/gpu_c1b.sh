cd $GRAFT_REPO_ROOT
for inf in 0 64 128; do
timeout 900 python tools/bench_configs.py c1d --rounds 12 --seq-rounds 12 --inflight $inf > gpurun_out/c1b_i$inf.log 2>&1; echo "inflight $inf rc=$?"
done
