cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_seq_levels.py tests/test_gpu_dense.py -q -x -s --timeout 600 > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/seq_epoch_time.py > gpurun_out/r2f_seqtime.log 2>&1; echo "time rc=$?"
timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > gpurun_out/r2f_c3_v2.log 2>&1; echo "c3v2 rc=$?"
