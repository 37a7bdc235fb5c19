cd $GRAFT_REPO_ROOT
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/turn_phases.py > gpurun_out/ph_n1.log 2>&1; echo "n1 rc=$?"
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n tools/turn_phases.py > gpurun_out/ph_n$n.log 2>&1; echo "n$n rc=$?"
done
