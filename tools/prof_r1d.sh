# Round-1d evidence (1 GPU, default bench): launch list, ncu --set full of the
# epoch, round turn, permutation and gap kernels, the L2 random-access ceiling.
CMD="python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_d.csv $CMD > gpurun_out/ncu1.log 2>&1
echo "launches rc=$?"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"scd_async|round_turn|hist2|scatter2|bsort2|colscan2" -s 12 -c 6 -o gpurun_out/prof_d $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
timeout 300 python tools/gap_bench.py > gpurun_out/gap_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:"gap_cols" -s 2 -c 1 -o gpurun_out/prof_gap python tools/gap_bench.py > gpurun_out/ncu_gap.log 2>&1
echo "gap rc=$?"
./tools/l2_random_roofline 100000 40000000 > gpurun_out/l2_roofline.json
echo "l2 rc=$?"
