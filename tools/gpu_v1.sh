cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/v1_tests.log 2>&1; echo "tests rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/v1_bench1.log 2>&1; echo "bench1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 > gpurun_out/v1_bench2.log 2>&1; echo "bench2 rc=$?"
