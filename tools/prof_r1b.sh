# Round-1 evidence for the default bench configuration (1 GPU):
#   plain run -> ncu launch list (cold, serialised; shares) -> ncu --set full of
#   the epoch kernel -> the L2 random-access ceiling microbenchmark.
CMD="python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
echo "launches rc=$?"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scd_async" -s 6 -c 1 \
  -o gpurun_out/prof_scd $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
./tools/l2_random_roofline 100000 40000000 > gpurun_out/l2_roofline.json
echo "l2 rc=$?"
