cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_engine.py tests/test_gpu_pipeline.py tests/test_gpu_dense.py -x -q > gpurun_out/conc_tests.log 2>&1; echo "tests rc=$?"
