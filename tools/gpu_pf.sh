cd $GRAFT_REPO_ROOT
B="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for pf in 0 1 2; do
  GLM_PERM_FORK=$pf timeout 300 $B > gpurun_out/pf${pf}_n1_$rep.log 2>&1; echo "n1 pf$pf rc=$?"
done; done
