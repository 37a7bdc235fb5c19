cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for cfg in "0 2" "1 1" "1 2" "0 1"; do
  set -- $cfg
  GLM_EPOCH_EARLY_TRIGGER=$1 GLM_TURN_BLOCKS_PER_SM=$2 CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/et2_e$1_tb$2_n1_$rep.log 2>&1; echo "n1 $cfg rc=$?"
  GLM_EPOCH_EARLY_TRIGGER=$1 GLM_TURN_BLOCKS_PER_SM=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/et2_e$1_tb$2_n4_$rep.log 2>&1; echo "n4 $cfg rc=$?"
done; done
