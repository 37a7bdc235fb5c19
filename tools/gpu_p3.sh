cd $GRAFT_REPO_ROOT
timeout 300 python tools/perm_time.py > gpurun_out/p3_perm_time.log 2>&1; echo "pt rc=$?"
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_pipeline.py tests/test_gpu_seq_levels.py -x -q > gpurun_out/p3_tests.log 2>&1; echo "tests rc=$?"
B="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 $B > gpurun_out/p3_n1_$rep.log 2>&1; echo "n1 rc=$?"
  timeout 300 $T > gpurun_out/p3_n2_$rep.log 2>&1; echo "n2 rc=$?"
done
GLM_PERM_FORK=2 CUDA_VISIBLE_DEVICES=0 timeout 300 $B > gpurun_out/p3_n1_pf2.log 2>&1; echo "n1 pf2 rc=$?"
