cd $GRAFT_REPO_ROOT
timeout 300 python tools/perm_bench.py 1000000 11000000 > gpurun_out/c3p_perm.log 2>&1; echo "perm rc=$?"
for pf in 0 2; do
GLM_PERM_FORK=$pf timeout 600 python tools/bench_multi.py c3 --rounds 6 > gpurun_out/c3p_pf$pf.log 2>&1; echo "c3 pf$pf rc=$?"
done
