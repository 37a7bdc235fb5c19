cd $GRAFT_REPO_ROOT
B="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for v in old new nodyn dyn; do
  cp abtest/$v.so paper_1803_06333_b200/libglm_b200.so
  timeout 300 $B > gpurun_out/ab3_${v}_$rep.log 2>&1; echo "$v rc=$?"
done; done
cp abtest/dyn.so paper_1803_06333_b200/libglm_b200.so
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_bench_config.py tests/test_gpu_solver.py tests/test_gpu_acceptance.py -x -q > gpurun_out/ab3_tests.log 2>&1; echo "tests rc=$?"
