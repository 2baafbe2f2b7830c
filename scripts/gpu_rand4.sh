# BASELINE configs[4]-style supremacy circuits on 4 GPUs (16 and 64 GiB per GPU)
cd $GRAFT_REPO_ROOT
for n in 32 34; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954${n: -1} \
  bench.py --gpus 4 --qubits $n --workload rand --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n4_rand$n.log 2>&1
echo "rc=$?" >> gpurun_out/bench_n4_rand$n.log
done
