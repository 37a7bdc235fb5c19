cd $GRAFT_REPO_ROOT
for k in 10 30 37; do
timeout 300 python bench.py --steps $k --warmup 3 --no-cpu --no-primal --no-ttt > gpurun_out/steps_k$k.log 2>&1; echo "k$k rc=$?"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29831 bench.py --gpus 2 --steps 30 --warmup 3 --no-cpu --no-primal --no-ttt > gpurun_out/steps_n2.log 2>&1; echo "n2 rc=$?"
