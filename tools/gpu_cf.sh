cd $GRAFT_REPO_ROOT
for cf in 1 3 2; do timeout 600 python tools/bench_configs.py c4 --rounds 6 --cache-flags $cf > gpurun_out/c4p_cf$cf.log 2>&1; echo "c4 packed cf$cf rc=$?"; done
for cf in 1 3 2 0; do timeout 300 python bench.py --steps 30 --warmup 5 --cache-flags $cf --no-primal > gpurun_out/c2_cf$cf.log 2>&1; echo "c2 cf$cf rc=$?"; done
