cd $GRAFT_REPO_ROOT
for cfg in "2 0" "1 0" "2 1" "1 1"; do
  set -- $cfg
  GLM_TURN_BLOCKS_PER_SM=$1 GLM_PEER_RS=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 tools/bench_multi.py c4 --rounds 6 > gpurun_out/c4x_tb$1_rs$2_n4.log 2>&1; echo "n4 $cfg rc=$?"
done
for cfg in "2" "1"; do
  GLM_TURN_BLOCKS_PER_SM=$cfg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 tools/bench_multi.py c4 --rounds 6 > gpurun_out/c4x_tb${cfg}_n2.log 2>&1; echo "n2 $cfg rc=$?"
done
