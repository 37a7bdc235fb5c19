cd $GRAFT_REPO_ROOT
for t in 3 6 20 60; do
SHARES=8 TRAJ=$t timeout 300 python tools/per_rank_epoch.py > gpurun_out/traj_t$t.log 2>&1; echo "t$t rc=$?"
done
