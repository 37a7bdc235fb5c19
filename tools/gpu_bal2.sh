cd $GRAFT_REPO_ROOT
for b in 0 1; do
GLM_EPOCH_BALANCE=$b SHARE=8 timeout 300 python tools/turn_phases.py > gpurun_out/bal2_ph_b$b.log 2>&1; echo "ph b$b rc=$?"
GLM_EPOCH_BALANCE=$b SHARE=8 TL_ROUNDS=3 timeout 300 python tools/round_timeline.py > gpurun_out/bal2_tl_b$b.log 2>&1; echo "tl b$b rc=$?"
done
