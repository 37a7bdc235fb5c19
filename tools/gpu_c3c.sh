cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_acceptance.py tests/test_gpu_restated.py -x -q > gpurun_out/c3c_tests.log 2>&1; echo "tests rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/bench_multi.py c3 --rounds 6 > gpurun_out/c3c_n1.log 2>&1; echo "c3 n1 rc=$?"
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2974$n tools/bench_multi.py c3 --rounds 6 > gpurun_out/c3c_n$n.log 2>&1; echo "c3 n$n rc=$?"
done
