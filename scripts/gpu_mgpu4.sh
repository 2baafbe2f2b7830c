# GPU tests + 4-GPU checks: rank-mode parity + benches (QAOA, rand) at N=4
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
  scripts/mgpu_check.py > gpurun_out/mgpu_check4.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/mgpu_check4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 \
  bench.py --gpus 4 --steps 3 --warmup 3 --workload qaoa --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n4_qaoa.log 2>&1
for n in 32 34; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954${n: -1} \
  bench.py --gpus 4 --qubits $n --workload rand --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n4_rand$n.log 2>&1
done
