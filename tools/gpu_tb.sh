cd $GRAFT_REPO_ROOT
B="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for tb in 2 1; do
  GLM_TURN_BLOCKS_PER_SM=$tb CUDA_VISIBLE_DEVICES=0 timeout 300 $B > gpurun_out/tb${tb}_n1_$rep.log 2>&1; echo "n1 tb$tb rc=$?"
  GLM_TURN_BLOCKS_PER_SM=$tb timeout 300 $T > gpurun_out/tb${tb}_n2_$rep.log 2>&1; echo "n2 tb$tb rc=$?"
done; done
for pf in 1 2; do
  GLM_PERM_FORK=$pf timeout 300 $T > gpurun_out/pf${pf}_n2.log 2>&1; echo "n2 pf$pf rc=$?"
done
