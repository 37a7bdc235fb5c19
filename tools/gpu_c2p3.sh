cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_restated.py tests/test_gpu_engine.py tests/test_gpu_solver.py tests/test_gpu_dense.py -x -q > gpurun_out/c2p3_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/bench_configs.py c2p --rounds 8 --seq-rounds 1 --no-cpu > gpurun_out/c2p3_auto.log 2>&1; echo "c2p rc=$?"
timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu --no-ttt > gpurun_out/c2p3_bench.log 2>&1; echo "bench rc=$?"
