cd $GRAFT_REPO_ROOT
for k in 4 8; do
VIRTUAL_NODES=$k timeout 900 python tools/async_vs_seq.py > gpurun_out/avs_k$k.log 2>&1; echo "k$k rc=$?"
done
