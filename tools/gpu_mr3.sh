cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_engine.py tests/test_gpu_bench_config.py tests/test_gpu_exchange.py -x -q > gpurun_out/mr3_tests.log 2>&1; echo "tests rc=$?"
B1="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for cfg in "x x" "0 2" "1 2"; do
  set -- $cfg
  if [ $1 = x ]; then E=""; else E="GLM_EPOCH_EARLY_TRIGGER=$1 GLM_TURN_BLOCKS_PER_SM=$2"; fi
  env $E CUDA_VISIBLE_DEVICES=0 timeout 300 $B1 > gpurun_out/mr3_e$1_tb$2_n1_$rep.log 2>&1; echo "n1 $cfg rc=$?"
done
for cfg in "x x" "0 2"; do
  set -- $cfg
  if [ $1 = x ]; then E=""; else E="GLM_EPOCH_EARLY_TRIGGER=$1 GLM_TURN_BLOCKS_PER_SM=$2"; fi
  for n in 2 4; do
  env $E timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/mr3_e$1_tb$2_n${n}_$rep.log 2>&1; echo "n$n $cfg rc=$?"
  done
done; done
