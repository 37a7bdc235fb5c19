cd $GRAFT_REPO_ROOT
./tools/view_ceiling 100000 40000000 > gpurun_out/r2b_view_ceiling.json 2>&1; echo "vc rc=$?"
./tools/view_ceiling 1000000 40000000 >> gpurun_out/r2b_view_ceiling.json 2>&1
timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > gpurun_out/r2b_c3.log 2>&1; echo "c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_replica" -s 2 -c 1 -o gpurun_out/r2b_c3_replica python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 3 --seq-rounds 0 > gpurun_out/r2b_ncu_c3.log 2>&1; echo "ncu rc=$?"
