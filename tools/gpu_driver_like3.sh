# What the driver runs at round end on a fresh 1-GPU box: the GPU suite,
# smoke(), the default bench line and the reference arm.
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/ -x -q -m gpu > gpurun_out/dl3_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dl3_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/dl3_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/dl3_ref.log 2>&1; echo "ref rc=$?"
