cd $GRAFT_REPO_ROOT
for et in 1 0; do
GLM_EPOCH_EARLY_TRIGGER=$et CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/bench_multi.py c4 --rounds 6 > gpurun_out/c4y_et${et}_n1.log 2>&1; echo "n1 et$et rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29573 tools/bench_multi.py c4 --rounds 6 > gpurun_out/c4y_n2.log 2>&1; echo "n2 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29574 tools/bench_multi.py c4 --rounds 6 > gpurun_out/c4y_n4.log 2>&1; echo "n4 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29575 bench.py --gpus 4 --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/c4y_c2n4.log 2>&1; echo "c2 n4 rc=$?"
