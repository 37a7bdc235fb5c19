cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_seq_levels.py tests/test_gpu_dense.py tests/test_gpu_restated.py -q -x -s --timeout 600 > gpurun_out/r2h_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/seq_epoch_time.py > gpurun_out/r2h_seqtime.log 2>&1; echo "time rc=$?"
timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > gpurun_out/r2h_c3_d1.log 2>&1; echo "c3d1 rc=$?"
GLM_NARROW_DELAY=2 timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > gpurun_out/r2h_c3_d2.log 2>&1; echo "c3d2 rc=$?"
for f in 2 4; do GLM_NARROW_DELAY=2 timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 --inflight $((3200*f)) > gpurun_out/r2h_c3_d2_b$f.log 2>&1; echo "c3d2b$f rc=$?"; done
