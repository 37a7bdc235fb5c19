cd $GRAFT_REPO_ROOT
PERM_NCU=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/p3_ncu.csv python tools/perm_time.py > gpurun_out/p3_ncu.log 2>&1; echo "ncu rc=$?"
PERM_NCU=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:region -s 2 -c 2 -o gpurun_out/p3_full python tools/perm_time.py > gpurun_out/p3_full.log 2>&1; echo "ncu full rc=$?"
