cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_exchange.py -x -q -k "two_process_exchange_matches" > gpurun_out/host_tests.log 2>&1; echo "tests rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2968$n bench.py --gpus $n --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/host_b$n.log 2>&1; echo "b$n rc=$?"
done
