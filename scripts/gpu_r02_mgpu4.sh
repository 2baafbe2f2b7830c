# QAOA-32@4: write-only budget 40 (round-1-like plan) vs the candidates
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02p4_build.log 2>&1
for b in 40 48 64 def; do
  if [ $b = def ]; then E="QS_X=0"; else E="QS_WO_BUDGET=$b"; fi
  env $E timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29900 + RANDOM % 90)) \
      bench.py --gpus 4 --steps 5 --warmup 3 --workload qaoa --e2e-steps 0 > gpurun_out/r02p4_qaoa_b$b.log 2>&1
done
