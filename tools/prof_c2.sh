set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits
CMD="python bench.py --steps 4 --warmup 3 --no-ttt --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scd_async|hist_kernel|scatter_kernel|bucket_sort|scan_kernel|value_kernel" -s 40 -c 6 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu2.log 2>&1
echo done $?
tail -3 gpurun_out/plain.log | cut -c1-300
