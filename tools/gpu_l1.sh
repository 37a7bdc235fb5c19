cd $GRAFT_REPO_ROOT
B="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for cfg in "1 1000" "17 1000" "1 0" "17 0" "16 0"; do
  set -- $cfg
  GLM_EPOCH_CARVEOUT=$2 timeout 300 $B --cache-flags $1 > gpurun_out/l1_cf$1_co$2_$rep.log 2>&1; echo "cf$1 co$2 rc=$?"
done; done
