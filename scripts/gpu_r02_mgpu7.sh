# QAOA at 2/4 GPUs with push/pull: write-only budget 64 vs the sharded default
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02r_build.log 2>&1
for N in 2 4; do
  DEV=$(seq -s, 0 $((N-1)))
  for b in def 64; do
    if [ $b = def ]; then E="QS_X=0"; else E="QS_WO_BUDGET=$b"; fi
    env $E CUDA_VISIBLE_DEVICES=$DEV QS_TIMING_DUMP=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29750 + N)) \
      bench.py --gpus $N --steps 3 --warmup 3 --workload qaoa --e2e-steps 0 > gpurun_out/r02r_qaoa_n${N}_b$b.log 2> gpurun_out/r02r_qaoa_n${N}_b$b.err
  done
done
