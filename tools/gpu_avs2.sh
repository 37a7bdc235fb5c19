cd $GRAFT_REPO_ROOT
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/async_vs_seq.py > gpurun_out/avs2_n1.log 2>&1; echo "n1 rc=$?"
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2982$n tools/async_vs_seq.py > gpurun_out/avs2_n$n.log 2>&1; echo "n$n rc=$?"
done
