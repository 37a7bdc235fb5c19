# launch list of a short bench run (cold-cache, serialised: compare shares)
CMD="python bench.py --steps 4 --warmup 3 --no-ttt --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
echo "ncu rc=$?"
