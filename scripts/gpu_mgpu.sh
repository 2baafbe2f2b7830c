# 2-GPU checks: rank-mode parity (NCCL swaps) + bench at N=2 (torchrun)
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  scripts/mgpu_check.py > gpurun_out/mgpu_check.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/mgpu_check.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2.log 2>&1
echo "bench2 rc=$?" >> gpurun_out/bench_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 2 --workload qaoa --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n2_qaoa.log 2>&1
