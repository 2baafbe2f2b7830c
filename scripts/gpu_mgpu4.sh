# 4-GPU: rank-mode parity + benches at N=4 and N=2 (QFT, QAOA, rand)
cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
  scripts/mgpu_check.py > gpurun_out/mgpu_check4.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/mgpu_check4.log
for G in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2952$G \
    bench.py --gpus $G --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n$G.log 2>&1
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2953$G \
    bench.py --gpus $G --steps 3 --warmup 3 --workload qaoa --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n${G}_qaoa.log 2>&1
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 \
  bench.py --gpus 4 --qubits 32 --workload rand --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n4_rand32.log 2>&1
