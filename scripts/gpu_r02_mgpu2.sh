# round 2 multi-GPU re-measure (gpurun --gpus 4): weak scaling 1/2/4 of the
# bench workloads with the final planner/kernels, rank-mode parity
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02n_build.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 \
  scripts/mgpu_check.py > gpurun_out/r02n_mgpu_check_n4.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/r02n_mgpu_check_n4.log
for N in 1 2 4; do
  DEV=$(seq -s, 0 $((N-1)))
  for wl in qft qaoa rand; do
    if [ $N = 1 ]; then
      CUDA_VISIBLE_DEVICES=$DEV timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02n_bench_n${N}_$wl.log 2>&1
    else
      CUDA_VISIBLE_DEVICES=$DEV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 297$N$((RANDOM % 9)) \
        bench.py --gpus $N --steps 5 --warmup 3 --workload $wl --e2e-steps 2 > gpurun_out/r02n_bench_n${N}_$wl.log 2>&1
    fi
  done
done
