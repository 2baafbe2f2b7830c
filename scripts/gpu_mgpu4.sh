# 4-GPU checks: rank-mode parity (NCCL swaps) + bench at N=4 and N=2 (torchrun)
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/topo4.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
  scripts/mgpu_check.py > gpurun_out/mgpu_check4.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/mgpu_check4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 \
  bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4.log 2>&1
echo "bench4 rc=$?" >> gpurun_out/bench_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29523 \
  bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 \
  bench.py --gpus 4 --steps 3 --warmup 3 --workload qaoa > gpurun_out/bench_n4_qaoa.log 2>&1
