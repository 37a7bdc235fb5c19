# Closing round-2 checks on one B200: smoke, the whole GPU suite, the default
# bench line and the reference arm.
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"
timeout 400 python bench.py > gpurun_out/final_b1.log 2>&1; echo "b1 rc=$?"
timeout 400 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?"
