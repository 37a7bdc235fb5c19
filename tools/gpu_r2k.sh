cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_exchange.py -q -x --timeout 600 > gpurun_out/r2k_exch.log 2>&1; echo "exch rc=$?"
GLM_LVL_DEBUG=1 timeout 300 python tools/seq_epoch_time.py 1 > gpurun_out/r2k_dbg.log 2>&1; echo "dbg rc=$?"
