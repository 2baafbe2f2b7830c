# QAOA-32@4 fused-pass A/B: multi-copy tensor loads on/off, repeated
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02o_build.log 2>&1
nvidia-smi topo -m > gpurun_out/r02o_topo.txt 2>&1
for rep in 1 2; do
  for tc in 1 64; do
    QS_JIT_TENSOR_COPIES=$tc timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800 + tc + rep)) \
      bench.py --gpus 4 --steps 5 --warmup 3 --workload qaoa --e2e-steps 0 > gpurun_out/r02o_qaoa_tc${tc}_r$rep.log 2>&1
  done
done
QS_NO_FUSED_SWAP=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29891 \
  bench.py --gpus 4 --steps 3 --warmup 3 --workload qaoa --e2e-steps 0 > gpurun_out/r02o_qaoa_nofuse.log 2>&1
