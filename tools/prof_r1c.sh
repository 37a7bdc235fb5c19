# Round-1c evidence (1 GPU, default bench): launch list, ncu --set full of the
# epoch kernel and of the round turn kernel, the L2 random-access ceiling.
CMD="python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c.csv $CMD > gpurun_out/ncu1.log 2>&1
echo "launches rc=$?"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"scd_async|round_turn" -s 8 -c 2 -o gpurun_out/prof_c $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
./tools/l2_random_roofline 100000 40000000 > gpurun_out/l2_roofline.json
echo "l2 rc=$?"
