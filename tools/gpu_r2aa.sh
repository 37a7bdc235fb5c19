cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu --no-primal > gpurun_out/r2aa_plain.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2aa_launches.csv python bench.py --steps 40 --warmup 3 --no-ttt --no-cpu --no-primal > gpurun_out/r2aa_ncu.log 2>&1; echo "ncu rc=$?"
