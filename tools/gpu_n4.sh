cd $GRAFT_REPO_ROOT
cp abtest/hack.so paper_1803_06333_b200/libglm_b200.so
for n in 1 2 4; do
for pf in 0 2 3; do
  if [ $n = 1 ]; then CUDA_VISIBLE_DEVICES=0 GLM_PERM_FORK=$pf timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/n4_pf${pf}_n$n.log 2>&1
  else GLM_PERM_FORK=$pf timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$pf bench.py --gpus $n --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/n4_pf${pf}_n$n.log 2>&1; fi
  echo "n$n pf$pf rc=$?"
done; done
