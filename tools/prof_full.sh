# ncu --set full of the epoch kernel of the default bench configuration (1 GPU)
CMD="python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu"
timeout 300 $CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scd_async" -s 6 -c 1 \
  -o gpurun_out/prof_scd $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
