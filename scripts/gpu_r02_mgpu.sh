# round 2 multi-GPU call (run with gpurun --gpus N): rank-mode parity, weak
# scaling benches with NVLink accounting, ncu NVLink counters of fused passes
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02m_build.log 2>&1
nvidia-smi topo -m > gpurun_out/r02m_topo.txt 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 \
  scripts/mgpu_check.py > gpurun_out/r02m_mgpu_check_n$N.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/r02m_mgpu_check_n$N.log
for wl in qft qaoa rand; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N \
    bench.py --gpus $N --steps 5 --warmup 3 --workload $wl --e2e-steps 2 > gpurun_out/r02m_bench_n${N}_$wl.log 2>&1
  QS_NO_FUSED_SWAP=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2963$N \
    bench.py --gpus $N --steps 3 --warmup 3 --workload $wl --e2e-steps 0 > gpurun_out/r02m_bench_n${N}_${wl}_nofuse.log 2>&1
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29641 \
  bench.py --impl reference --gpus $N --steps 2 --warmup 1 > gpurun_out/r02m_reference_n$N.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum \
  --clock-control none --csv --log-file gpurun_out/r02m_ncu_nvlink_qaoa_n2.csv python scripts/prof_mgpu.py qaoa 2 > gpurun_out/r02m_ncu_nvlink_qaoa.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02m_ncu_nvlink_qaoa.log
