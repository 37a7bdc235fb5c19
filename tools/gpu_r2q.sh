cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_seq_levels.py -q -x -s --timeout 600 > gpurun_out/r2q_lvl.log 2>&1; echo "lvl rc=$?"
timeout 600 python tools/seq_epoch_time.py > gpurun_out/r2q_seqtime.log 2>&1; echo "time rc=$?"
GLM_SEQ_KERNEL=lvl1 timeout 600 python tools/seq_epoch_time.py > gpurun_out/r2q_seqtime1.log 2>&1; echo "time1 rc=$?"
