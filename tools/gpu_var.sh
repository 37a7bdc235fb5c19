# Box-to-box spread of the default bench line (run once per fresh box).
cd $GRAFT_REPO_ROOT
TAG=${TAG:-x}
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu --no-primal > gpurun_out/var_${TAG}_b1.log 2>&1; echo "b1 rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2981$n bench.py --gpus $n > gpurun_out/var_${TAG}_b$n.log 2>&1; echo "b$n rc=$?"
done
nvidia-smi --query-gpu=name,serial,clocks.max.sm,power.limit --format=csv > gpurun_out/var_${TAG}_smi.csv 2>&1
