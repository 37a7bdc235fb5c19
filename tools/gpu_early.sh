cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_bench_config.py tests/test_gpu_engine.py -x -q > gpurun_out/early_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29781 tools/turn_phases.py > gpurun_out/early_ph4.log 2>&1; echo "ph4 rc=$?"
for rep in 1 2; do
for ea in 1 0; do
  for n in 2 4; do
  GLM_PEER_EARLY=$ea timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2979$n bench.py --gpus $n --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/early_e${ea}_n${n}_$rep.log 2>&1; echo "e$ea n$n rc=$?"
  done
done; done
