cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for lanes in 0 4 1288 8; do
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt --lanes $lanes > gpurun_out/lanes_l${lanes}_$rep.log 2>&1; echo "lanes $lanes rc=$?"
done; done
