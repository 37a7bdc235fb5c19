cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_pipeline.py -x -q > gpurun_out/ovf_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python tools/perm_time.py > gpurun_out/ovf_perm_time.log 2>&1; echo "pt rc=$?"
