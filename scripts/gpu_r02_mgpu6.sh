# push/pull split: loopback parity tests, rank-mode parity, QAOA/rand @4 A/B
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02q_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "loopback or sharded or fused" > gpurun_out/r02q_pytest_loopback.txt 2>&1
echo "rc=$?" >> gpurun_out/r02q_pytest_loopback.txt
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29731 \
  scripts/mgpu_check.py > gpurun_out/r02q_mgpu_check_n4.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/r02q_mgpu_check_n4.log
for wl in qaoa rand; do
  for np in 0 1; do
    if [ $np = 1 ]; then E="QS_NO_PULL=1"; else E="QS_X=0"; fi
    env $E QS_TIMING_DUMP=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29740 + np)) \
      bench.py --gpus 4 --steps 3 --warmup 3 --workload $wl --e2e-steps 0 > gpurun_out/r02q_${wl}_np$np.log 2> gpurun_out/r02q_${wl}_np$np.err
  done
done
