cd $GRAFT_REPO_ROOT
timeout 300 python tools/perm_time.py > gpurun_out/perm_time.log 2>&1; echo "pt rc=$?"
PERM_NCU=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/perm_ncu.csv python tools/perm_time.py > gpurun_out/perm_ncu.log 2>&1; echo "ncu rc=$?"
