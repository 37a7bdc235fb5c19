# Closing checks after the last parity additions: smoke, the whole
# GPU suite (4 GPUs visible), the default bench line at 1/2/4 GPUs, the
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f5_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/f5_tests.log 2>&1; echo "tests rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/f5_b1.log 2>&1; echo "b1 rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2985$n bench.py --gpus $n > gpurun_out/f5_b$n.log 2>&1; echo "b$n rc=$?"
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > gpurun_out/f5_ref.log 2>&1; echo "ref rc=$?"
