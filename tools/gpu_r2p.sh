cd $GRAFT_REPO_ROOT
timeout 400 python bench.py > gpurun_out/r2p_b1.log 2>&1; echo "b1 rc=$?"
