# 4-GPU checkpoint: the whole GPU suite (multi-GPU tests enabled), the bench at
# 1/2/4 GPUs, the reduce-scatter exchange on/off, C4 exchange, async contract.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2n_smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2n_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python bench.py > gpurun_out/r2n_b1.log 2>&1; echo "b1 rc=$?"
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n > gpurun_out/r2n_b$n.log 2>&1; echo "b$n rc=$?"
done
GLM_PEER_RS=0 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus 4 --no-ttt --no-cpu > gpurun_out/r2n_b4_nors.log 2>&1; echo "b4nors rc=$?"
for rs in 1 0; do
  GLM_PEER_RS=$rs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2963$rs tools/bench_multi.py c4 --rounds 6 > gpurun_out/r2n_c4_rs$rs.log 2>&1; echo "c4 rs$rs rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640 tools/async_vs_seq.py > gpurun_out/r2n_avs4.log 2>&1; echo "avs4 rc=$?"
