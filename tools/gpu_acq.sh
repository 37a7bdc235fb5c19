cd $GRAFT_REPO_ROOT
cp abtest/acq.so paper_1803_06333_b200/libglm_b200.so
timeout 1500 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_bench_config.py tests/test_gpu_engine.py -x -q > gpurun_out/acq_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29721 tools/turn_phases.py > gpurun_out/acq_ph4.log 2>&1; echo "ph4 rc=$?"
B1="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for v in sc acq; do
  cp abtest/$v.so paper_1803_06333_b200/libglm_b200.so
  CUDA_VISIBLE_DEVICES=0 timeout 300 $B1 > gpurun_out/acq_${v}_n1_$rep.log 2>&1; echo "$v n1 rc=$?"
  for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2973$n bench.py --gpus $n --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/acq_${v}_n${n}_$rep.log 2>&1; echo "$v n$n rc=$?"
  done
done; done
cp abtest/acq.so paper_1803_06333_b200/libglm_b200.so
