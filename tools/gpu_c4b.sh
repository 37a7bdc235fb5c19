cd $GRAFT_REPO_ROOT
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/bench_multi.py c4 --rounds 4 --breakdown > gpurun_out/c4b_n1.log 2>&1; echo "n1 rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n tools/bench_multi.py c4 --rounds 4 --breakdown > gpurun_out/c4b_n$n.log 2>&1; echo "n$n rc=$?"
done
