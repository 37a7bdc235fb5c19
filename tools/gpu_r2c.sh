cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_seq_levels.py -q -x -s --timeout 600 > gpurun_out/r2c_lvl.log 2>&1; echo "lvl rc=$?"
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/bench_configs.py c2 --rounds 14 --seq-rounds 14 > gpurun_out/r2c_c2modes.log 2>&1; echo "c2 rc=$?"
