cd $GRAFT_REPO_ROOT
for per in 1 2 4 8; do
GLM_NARROW_PER=$per timeout 900 python tools/bench_configs.py c3 --rounds 6 --seq-rounds 0 > gpurun_out/nper_p$per.log 2>&1; echo "per $per rc=$?"
done
