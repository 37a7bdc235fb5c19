cd $GRAFT_REPO_ROOT
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2968$n bench.py --gpus $n > gpurun_out/r2y_b$n.log 2>&1; echo "b$n rc=$?"
done
timeout 300 python bench.py > gpurun_out/r2y_b1.log 2>&1; echo "b1 rc=$?"
timeout 300 python bench.py --impl reference > gpurun_out/r2y_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 tools/hier_bench.py > gpurun_out/r2y_hier4.log 2>&1; echo "hier4 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 tools/bench_multi.py c3 --rounds 4 > gpurun_out/r2y_c3_4.log 2>&1; echo "c3x4 rc=$?"
