cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for rs in 0 1; do
GLM_PEER_RS=$rs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 4 --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/rs4_rs${rs}_$rep.log 2>&1; echo "rs$rs rc=$?"
done; done
GLM_PEER_RS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 tools/turn_phases.py > gpurun_out/rs4_ph.log 2>&1; echo "ph rc=$?"
