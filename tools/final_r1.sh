# Round-1 closing evidence: smoke, GPU tests, default bench at 1/2/4 GPUs, the
# reference arm, and the launch list of the default 1-GPU bench.
# (FINAL_QUICK=1: bench lines only)
if [ -z "$FINAL_QUICK" ]; then
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 420 python -m pytest tests -m gpu -q --timeout 90 > gpurun_out/gpu_all.log 2>&1; echo "tests rc=$?"
fi
timeout 300 python bench.py > gpurun_out/final_n1.log 2>&1; echo "n1 rc=$?"
timeout 300 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?"
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n > gpurun_out/final_n$n.log 2>&1; echo "n$n rc=$?"
done
if [ -z "$FINAL_QUICK" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_e.csv python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu > gpurun_out/ncu_e.log 2>&1; echo "ncu rc=$?"
fi
