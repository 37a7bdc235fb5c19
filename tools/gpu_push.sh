cd $GRAFT_REPO_ROOT
cp abtest/push.so paper_1803_06333_b200/libglm_b200.so
timeout 1500 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_bench_config.py -x -q > gpurun_out/push_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 tools/turn_phases.py > gpurun_out/push_ph4.log 2>&1; echo "ph4 rc=$?"
for rep in 1 2; do
for v in p3 push; do
  cp abtest/$v.so paper_1803_06333_b200/libglm_b200.so
  for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2966$n bench.py --gpus $n --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/push_${v}_n${n}_$rep.log 2>&1; echo "$v n$n rc=$?"
  done
done; done
cp abtest/push.so paper_1803_06333_b200/libglm_b200.so
