cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_seq_levels.py tests/test_gpu_exchange.py -q -x --timeout 600 > gpurun_out/r2j_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/seq_epoch_time.py > gpurun_out/r2j_seqtime.log 2>&1; echo "time rc=$?"
timeout 900 python tools/bench_configs.py c2p --rounds 30 --seq-rounds 2 > gpurun_out/r2j_c2p.log 2>&1; echo "c2p rc=$?"
timeout 600 python tools/bench_configs.py c1d --rounds 12 > gpurun_out/r2j_c1d.log 2>&1; echo "c1d rc=$?"
timeout 600 python tools/bench_configs.py c2cpu > gpurun_out/r2j_c2cpu.log 2>&1; echo "c2cpu rc=$?"
