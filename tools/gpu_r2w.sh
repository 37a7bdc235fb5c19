cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 tools/hier_bench.py > gpurun_out/r2w_hier4.log 2>&1; echo "hier4 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 tools/hier_bench.py > gpurun_out/r2w_hier2.log 2>&1; echo "hier2 rc=$?"
