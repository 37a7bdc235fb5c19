cd $GRAFT_REPO_ROOT
B1="python bench.py --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt"
for rep in 1 2; do
for v in cur e104_p5 e104_p6; do
  cp abtest/$v.so paper_1803_06333_b200/libglm_b200.so
  CUDA_VISIBLE_DEVICES=0 timeout 300 $B1 > gpurun_out/mr2_${v}_n1_$rep.log 2>&1; echo "$v n1 rc=$?"
  for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n bench.py --gpus $n --steps 40 --warmup 5 --no-cpu --no-primal --no-ttt > gpurun_out/mr2_${v}_n${n}_$rep.log 2>&1; echo "$v n$n rc=$?"
  done
done; done
for v in cur e104_p5; do
  cp abtest/$v.so paper_1803_06333_b200/libglm_b200.so
  CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/bench_multi.py c4 --rounds 6 > gpurun_out/mr2_c4_${v}.log 2>&1; echo "c4 $v rc=$?"
done
cp abtest/cur.so paper_1803_06333_b200/libglm_b200.so
