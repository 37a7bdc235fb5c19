cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_seq_lvl" -c 1 -o gpurun_out/r2g_lvl python tools/seq_epoch_time.py 1 > gpurun_out/r2g_ncu_lvl.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_replica" -c 1 -o gpurun_out/r2g_rep2 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 1 --seq-rounds 0 > gpurun_out/r2g_ncu_rep2.log 2>&1; echo "ncu2 rc=$?"
GLM_NARROW_KERNEL=v1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_replica" -c 1 -o gpurun_out/r2g_rep1 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 1 --seq-rounds 0 > gpurun_out/r2g_ncu_rep1.log 2>&1; echo "ncu3 rc=$?"
