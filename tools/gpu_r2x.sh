cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r2x_tests.log 2>&1; echo "tests rc=$?"
timeout 400 python bench.py --no-primal > gpurun_out/r2x_b1.log 2>&1; echo "b1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scd_async" -s 30 -c 1 -o gpurun_out/r2x_epoch python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu --no-primal > gpurun_out/r2x_ncu.log 2>&1; echo "ncu rc=$?"
