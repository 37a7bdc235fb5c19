cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in gapcur gap1 gap4 gap5; do
cp abtest/$v.so paper_1803_06333_b200/libglm_b200.so
timeout 300 python tools/gap_bench.py > gpurun_out/gapab_${v}_$rep.log 2>&1; echo "$v rc=$?"
done; done
cp abtest/gapcur.so paper_1803_06333_b200/libglm_b200.so
