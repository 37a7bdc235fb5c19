cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -x -k "exchange or bench_config" > gpurun_out/r2a_tests1.log 2>&1; echo "tests1 rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python bench.py > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?"
