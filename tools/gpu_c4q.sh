cd $GRAFT_REPO_ROOT
for nf in 1000000 250000; do
timeout 600 python tools/bench_configs.py c4 --rounds 6 --cache-flags 3 --n-feat $nf > gpurun_out/c4q_nf$nf.log 2>&1; echo "nf $nf rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sector_op_red_hit_rate.pct,dram__bytes_read.sum,lts__t_sectors.sum --clock-control none -k regex:"scd_async" -s 3 -c 1 python tools/bench_configs.py c4 --rounds 4 --cache-flags 3 --n-feat 250000 > gpurun_out/c4q_ncu250.log 2>&1; echo "ncu250 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sector_op_red_hit_rate.pct,dram__bytes_read.sum,lts__t_sectors.sum --clock-control none -k regex:"scd_async" -s 3 -c 1 python tools/bench_configs.py c4 --rounds 4 --cache-flags 3 > gpurun_out/c4q_ncu1m.log 2>&1; echo "ncu1m rc=$?"
