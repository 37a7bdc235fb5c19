cd $GRAFT_REPO_ROOT
timeout 300 python tools/perm_time.py > gpurun_out/p4_perm_time.log 2>&1; echo "pt rc=$?"
PERM_NCU=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/p4_ncu.csv python tools/perm_time.py > gpurun_out/p4_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_pipeline.py -x -q > gpurun_out/p4_tests.log 2>&1; echo "tests rc=$?"
B="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for v in old new new2; do
  cp abtest/$v.so paper_1803_06333_b200/libglm_b200.so
  timeout 300 $B > gpurun_out/ab2_${v}_$rep.log 2>&1; echo "$v rc=$?"
done; done
cp abtest/new2.so paper_1803_06333_b200/libglm_b200.so
