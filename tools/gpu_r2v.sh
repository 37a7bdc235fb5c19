cd $GRAFT_REPO_ROOT
for n in 1 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2965$n tools/turn_phases.py > gpurun_out/r2v_phases_$n.log 2>&1; echo "phases $n rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_exchange.py -q --timeout 600 > gpurun_out/r2v_tests.log 2>&1; echo "tests rc=$?"
