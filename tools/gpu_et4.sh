cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for et in x 1; do
  for n in 2 4; do
  if [ $et = x ]; then E=""; else E="GLM_EPOCH_EARLY_TRIGGER=$et"; fi
  env $E timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2976$n bench.py --gpus $n --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/et4_e${et}_n${n}_$rep.log 2>&1; echo "e$et n$n rc=$?"
  done
done; done
