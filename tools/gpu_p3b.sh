cd $GRAFT_REPO_ROOT
B="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 2 --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for cfg in "0 2" "1 2" "0 1" "1 1"; do
  set -- $cfg
  GLM_PERM_FORK=$1 GLM_TURN_BLOCKS_PER_SM=$2 CUDA_VISIBLE_DEVICES=0 timeout 300 $B > gpurun_out/p3b_pf$1_tb$2_n1_$rep.log 2>&1; echo "n1 $cfg rc=$?"
  GLM_PERM_FORK=$1 GLM_TURN_BLOCKS_PER_SM=$2 timeout 300 $T > gpurun_out/p3b_pf$1_tb$2_n2_$rep.log 2>&1; echo "n2 $cfg rc=$?"
done; done
