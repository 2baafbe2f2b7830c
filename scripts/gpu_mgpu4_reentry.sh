# 4-GPU re-entry check: rank-mode parity + QFT-32 / QAOA-32 benches at N=4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
  scripts/mgpu_check.py > gpurun_out/mgpu_check4.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/mgpu_check4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 \
  bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n4.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 4 --steps 3 --warmup 3 --workload qaoa --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n4_qaoa.log 2>&1
echo done
