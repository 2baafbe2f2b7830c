# round 2 final 4-GPU verification: rank-mode parity (with push/pull splits),
# weak scaling 1/2/4 of QFT/QAOA/rand through torchrun (driver-style)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f18_build.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 \
  scripts/mgpu_check.py > gpurun_out/r02f18_mgpu_check_n4.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/r02f18_mgpu_check_n4.log
for N in 2 4; do
  DEV=$(seq -s, 0 $((N-1)))
  for wl in qft qaoa rand; do
    CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29820 + N)) \
      bench.py --gpus $N --steps 5 --warmup 3 --workload $wl --e2e-steps 2 > gpurun_out/r02f18_bench_n${N}_$wl.log 2>&1
  done
  CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29830 + N)) \
      bench.py --impl reference --gpus $N --steps 2 --warmup 1 > gpurun_out/r02f18_reference_n$N.log 2>&1
done
