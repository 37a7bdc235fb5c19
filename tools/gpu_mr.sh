cd $GRAFT_REPO_ROOT
B1="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for v in cur mr104 mr112; do
  cp abtest/$v.so paper_1803_06333_b200/libglm_b200.so
  CUDA_VISIBLE_DEVICES=0 timeout 300 $B1 > gpurun_out/mr_${v}_n1_$rep.log 2>&1; echo "$v n1 rc=$?"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 4 --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/mr_${v}_n4_$rep.log 2>&1; echo "$v n4 rc=$?"
done; done
cp abtest/cur.so paper_1803_06333_b200/libglm_b200.so
