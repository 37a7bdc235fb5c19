cd $GRAFT_REPO_ROOT
GLM_LVL_DEBUG=1 timeout 300 python tools/seq_epoch_time.py 1 > gpurun_out/r2m_dbg.log 2>&1; echo "dbg rc=$?"
timeout 900 python -m pytest tests/test_gpu_acceptance.py -q -x -s --timeout 600 > gpurun_out/r2m_acc.log 2>&1; echo "acc rc=$?"
