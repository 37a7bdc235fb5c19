cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_exchange.py -q -x --timeout 600 > gpurun_out/r2l_exch.log 2>&1; echo "exch rc=$?"
GLM_LVL_DEBUG=1 timeout 300 python tools/seq_epoch_time.py 1 > gpurun_out/r2l_dbg.log 2>&1; echo "dbg rc=$?"
timeout 600 python tools/bench_multi.py c5 --n-per 8000000 --rounds 6 > gpurun_out/r2l_c5.log 2>&1; echo "c5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_async" -s 4 -c 1 -o gpurun_out/r2l_c5_train python tools/bench_configs.py c5 --n 8000000 --budget-gb 8 --epochs 2 > gpurun_out/r2l_ncu_c5.log 2>&1; echo "ncu rc=$?"
