cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_seq_levels.py -q -x -s --timeout 600 > gpurun_out/r2s_lvl.log 2>&1; echo "lvl rc=$?"
timeout 600 python tools/seq_determinism.py 8 1 > gpurun_out/r2s_det.log 2>&1; echo "det rc=$?"
timeout 600 python tools/seq_epoch_time.py > gpurun_out/r2s_seqtime.log 2>&1; echo "time rc=$?"
GLM_LVL_DEBUG=1 timeout 300 python tools/seq_epoch_time.py 1 > gpurun_out/r2s_dbg.log 2>&1; echo "dbg rc=$?"
