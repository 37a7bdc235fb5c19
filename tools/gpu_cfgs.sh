# Closing refresh of the other BASELINE configs at 1/2/4 GPUs (bench_multi: C3,
# C4, C5) and the 1-GPU configs (bench_configs: C1 dual, C2 primal).
cd $GRAFT_REPO_ROOT
O=gpurun_out/cfgs_multi.jsonl
rm -f $O
for c in c3 c4 c5; do
  CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/bench_multi.py $c --rounds 6 --out $O > gpurun_out/cfgs_${c}_n1.log 2>&1; echo "$c n1 rc=$?"
  for n in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n tools/bench_multi.py $c --rounds 6 --out $O > gpurun_out/cfgs_${c}_n$n.log 2>&1; echo "$c n$n rc=$?"
  done
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/bench_configs.py c1d > gpurun_out/cfgs_c1d.log 2>&1; echo "c1d rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/bench_configs.py c2p --no-cpu > gpurun_out/cfgs_c2p.log 2>&1; echo "c2p rc=$?"
