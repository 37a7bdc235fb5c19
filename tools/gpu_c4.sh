cd $GRAFT_REPO_ROOT
for cf in 0 1 2 3; do timeout 600 python tools/bench_configs.py c4 --rounds 6 --cache-flags $cf > gpurun_out/c4_cf$cf.log 2>&1; echo "c4 cf$cf rc=$?"; done
