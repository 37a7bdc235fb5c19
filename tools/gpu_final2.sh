# Closing checks after the permutation / turn-shape changes: smoke, the whole
# GPU suite (4 GPUs visible), the default bench line at 1/2/4 GPUs, the
# reference arm, and the launch list of the bench's timed rounds.
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/f2_tests.log 2>&1; echo "tests rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/f2_b1.log 2>&1; echo "b1 rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n bench.py --gpus $n > gpurun_out/f2_b$n.log 2>&1; echo "b$n rc=$?"
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > gpurun_out/f2_ref.log 2>&1; echo "ref rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu --no-primal > gpurun_out/f2_ncu.log 2>&1; echo "ncu rc=$?"
