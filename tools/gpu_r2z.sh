cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x --timeout 600 > gpurun_out/r2z_dense.log 2>&1; echo "dense rc=$?"
timeout 600 python tools/bench_configs.py c1d --rounds 12 --no-cpu > gpurun_out/r2z_c1d.log 2>&1; echo "c1d rc=$?"
timeout 600 python tools/bench_configs.py c1 --rounds 6 > gpurun_out/r2z_c1.log 2>&1; echo "c1 rc=$?"
timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > gpurun_out/r2z_c3.log 2>&1; echo "c3 rc=$?"
