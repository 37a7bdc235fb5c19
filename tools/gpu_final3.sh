# Closing checks after the register budget and turn changes: smoke, the whole
# GPU suite (4 GPUs visible), the default bench line at 1/2/4 GPUs, the
# reference arm, the launch list, and ncu --set full of one epoch launch.
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/f3_tests.log 2>&1; echo "tests rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/f3_b1.log 2>&1; echo "b1 rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n > gpurun_out/f3_b$n.log 2>&1; echo "b$n rc=$?"
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > gpurun_out/f3_ref.log 2>&1; echo "ref rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f3_launches.csv python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu --no-primal > gpurun_out/f3_ncu.log 2>&1; echo "ncu rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scd_async" -s 30 -c 1 -o gpurun_out/f3_epoch python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu --no-primal > gpurun_out/f3_ncufull.log 2>&1; echo "ncu full rc=$?"
