cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_exchange.py -q -x --timeout 600 > gpurun_out/r2i_exch.log 2>&1; echo "exch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_seq_lvl" -c 1 -o gpurun_out/r2i_lvl python tools/seq_epoch_time.py 1 > gpurun_out/r2i_ncu_lvl.log 2>&1; echo "ncu rc=$?"
for env in "GLM_NARROW_KERNEL=v1" "GLM_NARROW_KERNEL=v2" "GLM_NARROW_KERNEL=v2 GLM_NARROW_DELAY=2"; do
  env $env timeout 300 python tools/bench_configs.py c3 --n 11000000 --lam 100 --rounds 4 --seq-rounds 0 > "gpurun_out/r2i_c3_$(echo $env | tr ' =' '__').log" 2>&1; echo "c3 $env rc=$?"
done
