cd $GRAFT_REPO_ROOT
df -hT . /tmp > gpurun_out/r2t_df.txt 2>&1; free -g >> gpurun_out/r2t_df.txt
timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -x -s --timeout 600 > gpurun_out/r2t_pipe.log 2>&1; echo "pipe rc=$?"
timeout 900 python tools/disk_stream.py 8000000 > gpurun_out/r2t_disk.log 2>&1; echo "disk rc=$?"
