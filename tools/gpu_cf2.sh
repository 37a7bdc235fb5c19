cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for cf in 1 0; do
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt --cache-flags $cf > gpurun_out/cf2_c${cf}_$rep.log 2>&1; echo "cf$cf rc=$?"
done; done
