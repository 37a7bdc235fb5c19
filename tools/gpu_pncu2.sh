cd $GRAFT_REPO_ROOT
PERM_NCU=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:region -s 2 -c 2 -o gpurun_out/p5_full python tools/perm_time.py > gpurun_out/p5_full.log 2>&1; echo "ncu full rc=$?"
