cd $GRAFT_REPO_ROOT
B="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for et in 0 1; do
  GLM_EPOCH_EARLY_TRIGGER=$et CUDA_VISIBLE_DEVICES=0 timeout 300 $B > gpurun_out/et${et}_n1_$rep.log 2>&1; echo "n1 et$et rc=$?"
  GLM_EPOCH_EARLY_TRIGGER=$et timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/et${et}_n2_$rep.log 2>&1; echo "n2 et$et rc=$?"
done; done
for et in 0 1; do
  GLM_EPOCH_EARLY_TRIGGER=$et CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/turn_phases.py > gpurun_out/et${et}_ph1.log 2>&1; echo "ph1 et$et rc=$?"
  GLM_EPOCH_EARLY_TRIGGER=$et timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/turn_phases.py > gpurun_out/et${et}_ph2.log 2>&1; echo "ph2 et$et rc=$?"
done
