# 2-GPU re-entry check: GPU tests with 2 devices, rank-mode parity, bench at N=2 (qft, qaoa)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  scripts/mgpu_check.py > gpurun_out/mgpu_check.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/mgpu_check.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2.log 2>&1
echo "bench2 rc=$?" >> gpurun_out/bench_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 2 --workload qaoa --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n2_qaoa.log 2>&1
echo "bench2q rc=$?" >> gpurun_out/bench_n2_qaoa.log
