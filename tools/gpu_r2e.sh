cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_seq_lvl" -c 1 -o gpurun_out/r2e_lvl python tools/seq_epoch_time.py 1 > gpurun_out/r2e_ncu_lvl.log 2>&1; echo "ncu rc=$?"
timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > gpurun_out/r2e_c3_v2.log 2>&1; echo "c3v2 rc=$?"
GLM_NARROW_KERNEL=v1 timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > gpurun_out/r2e_c3_v1.log 2>&1; echo "c3v1 rc=$?"
timeout 600 python -m pytest tests/test_gpu_dense.py -q -x --timeout 300 > gpurun_out/r2e_dense.log 2>&1; echo "dense rc=$?"
