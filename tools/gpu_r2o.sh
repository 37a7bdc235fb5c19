cd $GRAFT_REPO_ROOT
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_seq.py > gpurun_out/r2o_san_$tool.log 2>&1; echo "$tool rc=$?"
done
timeout 300 python bench.py --no-ttt --no-cpu --steps 200 > gpurun_out/r2o_b1.log 2>&1; echo "b1 rc=$?"
GLM_TURN_BLOCKS_PER_SM=1 timeout 300 python bench.py --no-ttt --no-cpu --steps 200 > gpurun_out/r2o_b1_t1.log 2>&1; echo "b1t1 rc=$?"
