cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for b in 0 1; do
GLM_EPOCH_BALANCE=$b timeout 600 python tools/per_rank_epoch.py > gpurun_out/bal_b${b}_$rep.log 2>&1; echo "b$b rc=$?"
done; done
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_bench_config.py -x -q > gpurun_out/bal_tests.log 2>&1; echo "tests rc=$?"
