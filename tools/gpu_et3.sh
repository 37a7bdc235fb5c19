cd $GRAFT_REPO_ROOT
run() {  # e tb n rep
  if [ $3 = 1 ]; then GLM_EPOCH_EARLY_TRIGGER=$1 GLM_TURN_BLOCKS_PER_SM=$2 CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/et3_e$1_tb$2_n$3_$4.log 2>&1
  else GLM_EPOCH_EARLY_TRIGGER=$1 GLM_TURN_BLOCKS_PER_SM=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $3 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $3 --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/et3_e$1_tb$2_n$3_$4.log 2>&1; fi
  echo "e$1 tb$2 n$3 rc=$?"
}
for rep in 1 2 3; do
  for n in 1 2 4; do
    run 1 1 $n $rep
    run 0 1 $n $rep
    run 0 2 $n $rep
  done
done
