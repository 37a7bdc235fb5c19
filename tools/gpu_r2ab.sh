cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_bench_config.py -q -x --timeout 600 > gpurun_out/r2ab_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python bench.py --no-ttt --no-cpu --no-primal --steps 200 > gpurun_out/r2ab_b1.log 2>&1; echo "b1 rc=$?"
timeout 300 python tools/turn_phases.py > gpurun_out/r2ab_phases1.log 2>&1; echo "ph rc=$?"
