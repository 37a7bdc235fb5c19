cd $GRAFT_REPO_ROOT
timeout 300 python tools/round_timeline.py > gpurun_out/tl1.log 2>&1; echo "tl1 rc=$?"
TL_ROUNDS=3 timeout 300 python tools/round_timeline.py > gpurun_out/tl3.log 2>&1; echo "tl3 rc=$?"
