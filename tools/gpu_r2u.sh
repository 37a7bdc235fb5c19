cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x --timeout 600 > gpurun_out/r2u_dense.log 2>&1; echo "dense rc=$?"
timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > gpurun_out/r2u_c3_v1.log 2>&1; echo "c3 rc=$?"
GLM_NARROW_KERNEL=cl timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > gpurun_out/r2u_c3_cl.log 2>&1; echo "c3cl rc=$?"
for f in 2 4; do GLM_NARROW_KERNEL=cl timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 --inflight $((3200*f)) > gpurun_out/r2u_c3_cl_b$f.log 2>&1; echo "c3cl b$f rc=$?"; done
