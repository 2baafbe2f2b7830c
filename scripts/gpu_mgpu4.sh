# GPU tests + 4-GPU checks: rank-mode parity (NCCL / fused swaps) + QAOA benches at N=4 and N=2
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
  scripts/mgpu_check.py > gpurun_out/mgpu_check4.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/mgpu_check4.log
for G in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2952$G \
  bench.py --gpus $G --steps 3 --warmup 3 --workload qaoa --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n${G}_qaoa.log 2>&1
QS_NO_FUSED_SWAP=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2953$G \
  bench.py --gpus $G --steps 3 --warmup 3 --workload qaoa --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n${G}_qaoa_nofuse.log 2>&1
done
