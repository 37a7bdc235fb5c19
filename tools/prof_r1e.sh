# Round-1 closing ncu capture (1 GPU): epoch + turn kernels of the default bench.
CMD="python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu"
timeout 300 $CMD > gpurun_out/plain_e.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"scd_async|round_turn" -s 12 -c 2 -o gpurun_out/prof_e $CMD > gpurun_out/ncu_full_e.log 2>&1
echo "full rc=$?"
