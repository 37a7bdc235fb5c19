cd $GRAFT_REPO_ROOT
B="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2 3; do
for v in old new; do
  cp abtest/$v.so paper_1803_06333_b200/libglm_b200.so
  timeout 300 $B > gpurun_out/ab_${v}_$rep.log 2>&1; echo "$v rc=$?"
done; done
