# QAOA-32@4 per-launch timings of the 40- and 64-budget plans
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02p5_build.log 2>&1
for b in 40 64; do
  QS_TIMING_DUMP=1 QS_WO_BUDGET=$b timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29900 + b)) \
      bench.py --gpus 4 --steps 1 --warmup 3 --workload qaoa --e2e-steps 0 > gpurun_out/r02p5_qaoa_b$b.log 2> gpurun_out/r02p5_qaoa_b$b.err
done
