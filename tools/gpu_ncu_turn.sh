cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"round_turn" -s 30 -c 1 -o gpurun_out/turn_full python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu --no-primal > gpurun_out/turn_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"region_" -s 60 -c 2 -o gpurun_out/perm_full python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu --no-primal > gpurun_out/perm_ncu.log 2>&1; echo "ncu2 rc=$?"
