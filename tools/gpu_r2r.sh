cd $GRAFT_REPO_ROOT
timeout 600 python tools/seq_determinism.py 8 1 > gpurun_out/r2r_det.log 2>&1; echo "det rc=$?"
timeout 900 python -m pytest tests/test_gpu_seq_levels.py -q -x -s --timeout 600 > gpurun_out/r2r_lvl.log 2>&1; echo "lvl rc=$?"
